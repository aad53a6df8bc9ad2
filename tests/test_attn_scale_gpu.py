"""Bench-scale parity of K1 (forward) and K2 (backward) at the shapes the
step and the c5 sweep actually run — 16K-32K query slices, 32-64 heads,
8-32 KV chunks scattered in the arena, and a 1M-key prefix — on sampled
heads, query rows and key rows against the fp64 oracle
(oracle/attention_oracle.c orc_fwd_rows / orc_bwd_rows / orc_bwd_keys, the
reference fold attention.cpp:21-111 and the exact backward).

Full-size CPU oracles are infeasible (one c2 slice-8 head is ~0.5 TFLOP of
fp64 work), so the inputs are generated on the GPU from a seeded generator,
the whole slice runs through the kernels, and only the sampled heads come
back to the host.  The backward is checked as the function the kernel
implements, of (Q, K, V, O, dO, LSE) with the forward's O / LSE as inputs;
those are pinned on the same sampled rows by the forward check.

Tolerances (north_star "rel 2e-2 bf16"): O rel 2e-2 with the reference's
max(1, |ref|) denominator; LSE abs 2e-3; gradients per sampled row / key
max|g - ref| <= 2e-2 * max|ref| of that row (stricter than per tensor).
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle_lib as O
from test_attn_gpu import _need_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
TOL_O, TOL_LSE, TOL_G = 2e-2, 2e-3, 2e-2
D = 128

# name, slice rows Ls, heads, kv heads, chunks, chunk length, sampled heads
CASES = [
    ("c2_slice8", 16384, 32, 32, 8, 16384, (0, 17, 31)),        # c2: last of 8 slices, 128K keys
    ("c5_prefix1M", 16384, 32, 32, 1, 16384 + (1 << 20), (3,)),  # c5: 1M prefix + diagonal as one chunk
    ("c4_gqa_slice32", 32768, 64, 8, 32, 32768, (0, 7, 63)),   # c4: GQA 64/8, last of 32 slices, 1M keys
]


def _rows_sample(Ls, rng):
    fixed = [0, 1, 127, 128, Ls // 2, Ls - 2, Ls - 1]
    return np.unique(np.concatenate([fixed, rng.integers(0, Ls, 9)])).astype(np.int32)


def _keys_sample(n, L, rng):
    T = n * L
    fixed = [0, L - 1, (n // 2) * L, T - L, T - L // 2, T - 1]
    return np.unique(np.concatenate([fixed, rng.integers(0, T, 12)])).astype(np.int32)


def _rowwise_err(g, r):
    g, r = np.asarray(g, np.float64), np.asarray(r, np.float64)
    return float(np.max(np.max(np.abs(g - r), axis=1) / np.maximum(1e-30, np.max(np.abs(r), axis=1))))


@pytest.mark.parametrize("name,Ls,heads,kv,n,L,hs", CASES, ids=[c[0] for c in CASES])
def test_attention_at_bench_scale_matches_oracle(name, Ls, heads, kv, n, L, hs):
    _need_gpu()
    from paper_2504_14519_b200 import ops
    gen = torch.Generator(device="cuda").manual_seed(20240817)  # kernel seed, reference verify.hpp:22
    rng = np.random.default_rng(7)
    uni = lambda *s: (torch.rand(*s, device="cuda", generator=gen, dtype=torch.float32) * 2 - 1).bfloat16()
    qd, kvd, T = heads * D, kv * D, n * L
    # chunks in attention order 1..n live in shuffled arena slots (one spare)
    slots = [int(x) for x in rng.permutation(n + 1)[:n]] if n > 1 else [0]
    pool_rows = (max(slots) + 1) * L
    kp = torch.zeros(pool_rows, kvd, device="cuda", dtype=torch.bfloat16)
    vp = torch.zeros_like(kp)
    for c in range(n):  # generated in attention order so the oracle view is a plain concatenation
        kp[slots[c] * L:(slots[c] + 1) * L] = uni(L, kvd)
        vp[slots[c] * L:(slots[c] + 1) * L] = uni(L, kvd)
    rows_tab = [s * L for s in slots]
    q, do = uni(Ls, qd), uni(Ls, qd)
    o, lse = ops.attn_fwd(q, kp, vp, rows_tab, L, heads, kv, True)
    dq = torch.zeros(Ls, qd, device="cuda")
    dk = torch.zeros(pool_rows, kvd, device="cuda")
    dv = torch.zeros_like(dk)
    ops.attn_bwd(q, kp, vp, rows_tab, L, heads, kv, True, o, lse, do, dq, dk, dv, rows_tab)
    torch.cuda.synchronize()

    rsel, ksel = _rows_sample(Ls, rng), _keys_sample(n, L, rng)
    in_order = lambda pool, g: torch.cat([pool[s * L:(s + 1) * L, g * D:(g + 1) * D] for s in slots]).float().cpu().numpy()
    report = []
    for h in hs:
        g = h // (heads // kv)
        col = slice(h * D, (h + 1) * D)
        qh, oh, doh = (x[:, col].float().cpu().numpy() for x in (q, o, do))
        kh, vh = in_order(kp, g), in_order(vp, g)
        lse_h = lse[h].double().cpu().numpy()
        # forward: sampled rows
        ro, rl = O.port_fwd_rows(qh, kh, vh, True, rsel)
        # O: the reference's max(1,|x|) metric is near-vacuous when a row
        # averages 1M random values (|O| ~ 1e-3), so also row-relative
        e_o = max(float(np.max(np.abs(oh[rsel] - ro) / np.maximum(1.0, np.abs(ro)))), _rowwise_err(oh[rsel], ro))
        e_l = float(np.max(np.abs(lse_h[rsel] - rl)))
        # backward: dQ rows (this head) and dK/dV keys (this head's share)
        rdq = O.port_bwd_rows(qh, kh, vh, oh, doh, lse_h, True, rsel)
        e_dq = _rowwise_err(dq[:, col].cpu().numpy()[rsel], rdq)
        grp = range(g * (heads // kv), (g + 1) * (heads // kv))
        rdk, rdv = np.zeros((len(ksel), D)), np.zeros((len(ksel), D))
        for hh in grp:  # dK/dV of a kv head sum over its query heads (GQA)
            colh = slice(hh * D, (hh + 1) * D)
            a, b = O.port_bwd_keys(q[:, colh].float().cpu().numpy(), kh, vh, o[:, colh].float().cpu().numpy(),
                                   do[:, colh].float().cpu().numpy(), lse[hh].double().cpu().numpy(), True, ksel)
            rdk += a
            rdv += b
        gdk, gdv = in_order(dk, g)[ksel], in_order(dv, g)[ksel]
        e_dk, e_dv = _rowwise_err(gdk, rdk), _rowwise_err(gdv, rdv)
        report.append((h, e_o, e_l, e_dq, e_dk, e_dv))
        print(f"{name} head {h}: O {e_o:.2e} LSE {e_l:.2e} dQ {e_dq:.2e} dK {e_dk:.2e} dV {e_dv:.2e}")
    for h, e_o, e_l, e_dq, e_dk, e_dv in report:
        assert e_o < TOL_O and e_l < TOL_LSE, (name, h, e_o, e_l)
        assert e_dq < TOL_G and e_dk < TOL_G and e_dv < TOL_G, (name, h, e_dq, e_dk, e_dv)
