"""GPU parity of the attention backward kernel (K2) against the fp64 oracle.

The oracle gradients (oracle/attention_oracle.c:orc_attn_bwd_head) are pinned
to the reference forward by finite differences in tests/test_oracle.py.
Tolerance: the kernel feeds bf16 P and dS to the tensor cores (fp32
accumulation), so gradients are compared with a bf16-level bound,
max|gpu - oracle| <= 2e-2 * max|oracle| per tensor ("parity").
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle_lib as O
from test_attn_gpu import _need_gpu, bf16_round

pytestmark = pytest.mark.gpu
TOL = 2e-2


def nerr(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(1e-30, np.max(np.abs(b))))


def _t(x, dtype=torch.bfloat16):
    return torch.from_numpy(np.ascontiguousarray(x.reshape(x.shape[0], -1), dtype=np.float32)).cuda().to(dtype)


def _run_slices(q_all, k, v, do_all, L, heads, kv_heads, order):
    """Emulate the step: backward of slices n..1, slice i attending chunks 1..i,
    with K/V and the dK/dV accumulators in shuffled pool slots."""
    from paper_2504_14519_b200 import ops
    n = k.shape[0] // L
    d = q_all.shape[-1]
    pool_rows = (max(order) + 1) * L
    kp = np.zeros((pool_rows,) + k.shape[1:], np.float32)
    vp = np.zeros_like(kp)
    for c, slot in enumerate(order):
        kp[slot * L:(slot + 1) * L] = k[c * L:(c + 1) * L]
        vp[slot * L:(slot + 1) * L] = v[c * L:(c + 1) * L]
    kpt, vpt = _t(kp), _t(vp)
    dk_acc = torch.zeros(pool_rows, kv_heads * d, device="cuda")
    dv_acc = torch.zeros_like(dk_acc)
    dq_out = np.zeros_like(q_all, dtype=np.float64)
    for i in range(n, 0, -1):
        q = q_all[(i - 1) * L:i * L]
        do = do_all[(i - 1) * L:i * L]
        rows = [order[c] * L for c in range(i)]
        qt, dot = _t(q), _t(do)
        o, lse = ops.attn_fwd(qt, kpt, vpt, rows, L, heads, kv_heads, True, head_dim=d)
        dq = torch.zeros(L, heads * d, device="cuda")
        ops.attn_bwd(qt, kpt, vpt, rows, L, heads, kv_heads, True, o, lse, dot, dq, dk_acc, dv_acc, rows,
                     delta_ws=torch.empty(2 * heads * L, device="cuda"))
        torch.cuda.synchronize()
        dq_out[(i - 1) * L:i * L] = dq.cpu().numpy().reshape(L, heads, d)
    dk = dk_acc.cpu().numpy().reshape(pool_rows, kv_heads, d)
    dv = dv_acc.cpu().numpy().reshape(pool_rows, kv_heads, d)
    dk = np.concatenate([dk[order[c] * L:(order[c] + 1) * L] for c in range(n)])
    dv = np.concatenate([dv[order[c] * L:(order[c] + 1) * L] for c in range(n)])
    return dq_out, dk, dv


def _oracle_slices(q_all, k, v, do_all, L, n):
    """Sum over slices of the per-slice oracle gradients (forward O/lse from the oracle)."""
    dq = np.zeros(q_all.shape)
    dk = np.zeros(k.shape)
    dv = np.zeros(v.shape)
    for i in range(1, n + 1):
        q = q_all[(i - 1) * L:i * L]
        do = do_all[(i - 1) * L:i * L]
        _, lse = O.port_mha_fwd(q, k[:i * L], v[:i * L], [L] * i, True)
        a, b, c = O.port_mha_bwd(q, k[:i * L], v[:i * L], do, lse, True)
        dq[(i - 1) * L:i * L] += a
        dk[:i * L] += b
        dv[:i * L] += c
    return dq, dk, dv


@pytest.mark.parametrize("d,heads,kv_heads,n,L", [
    (128, 2, 2, 1, 128),
    (128, 2, 2, 3, 128),
    (128, 4, 1, 2, 256),   # GQA 4:1
    (64, 4, 4, 4, 128),    # c1 head_dim, 4 slices
    (64, 2, 1, 2, 256),
])
def test_bwd_sliced_accumulation_matches_oracle(d, heads, kv_heads, n, L):
    _need_gpu()
    rng = np.random.default_rng(300 + d * heads + n)
    S = n * L
    q = bf16_round(rng.uniform(-1, 1, (S, heads, d)))
    k = bf16_round(rng.uniform(-1, 1, (S, kv_heads, d)))
    v = bf16_round(rng.uniform(-1, 1, (S, kv_heads, d)))
    do = bf16_round(rng.uniform(-1, 1, (S, heads, d)))
    order = list(rng.permutation(n + 1)[:n])
    g_dq, g_dk, g_dv = _run_slices(q, k, v, do, L, heads, kv_heads, [int(x) for x in order])
    r_dq, r_dk, r_dv = _oracle_slices(q, k, v, do, L, n)
    assert nerr(g_dq, r_dq) < TOL
    assert nerr(g_dk, r_dk) < TOL
    assert nerr(g_dv, r_dv) < TOL


def test_bwd_non_causal_single_call():
    _need_gpu()
    from paper_2504_14519_b200 import ops
    rng = np.random.default_rng(5)
    d, heads, L, n = 128, 2, 128, 2
    q = bf16_round(rng.uniform(-1, 1, (L, heads, d)))
    k = bf16_round(rng.uniform(-1, 1, (n * L, heads, d)))
    v = bf16_round(rng.uniform(-1, 1, (n * L, heads, d)))
    do = bf16_round(rng.uniform(-1, 1, (L, heads, d)))
    _, lse = O.port_mha_fwd(q, k, v, [L] * n, False)
    r_dq, r_dk, r_dv = O.port_mha_bwd(q, k, v, do, lse, False)
    qt, kt, vt, dot = _t(q), _t(k), _t(v), _t(do)
    o, lse_g = ops.attn_fwd(qt, kt, vt, [0, L], L, heads, heads, False)
    dq = torch.zeros(L, heads * d, device="cuda")
    dk = torch.zeros(n * L, heads * d, device="cuda")
    dv = torch.zeros_like(dk)
    ops.attn_bwd(qt, kt, vt, [0, L], L, heads, heads, False, o, lse_g, dot, dq, dk, dv, [0, L],
                 delta_ws=torch.empty(2 * heads * L, device="cuda"))
    torch.cuda.synchronize()
    assert nerr(dq.cpu().numpy().reshape(q.shape), r_dq) < TOL
    assert nerr(dk.cpu().numpy().reshape(k.shape), r_dk) < TOL
    assert nerr(dv.cpu().numpy().reshape(v.shape), r_dv) < TOL
