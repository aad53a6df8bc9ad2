"""torch-tensor front end of the device C-ABI (include/slimpipe.h).

Thin plumbing: validates dtypes/devices, passes data pointers and the current
CUDA stream to libslimpipe.so.  The math lives in the sm_100a kernels; there
is no torch fallback — a missing library or an unsupported shape raises.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import native as N


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: torch.Tensor | None):
    return C.c_void_p(t.data_ptr() if t is not None else 0)


def _rows(chunk_rows):
    vals = [int(x) for x in chunk_rows]
    return (C.c_int32 * max(1, len(vals)))(*vals), len(vals)


def attn_fwd(q: torch.Tensor, k_pool: torch.Tensor, v_pool: torch.Tensor, chunk_rows, chunk_len: int, heads: int,
             kv_heads: int, causal: bool = True, o: torch.Tensor | None = None, lse: torch.Tensor | None = None,
             head_dim: int | None = None):
    """Sliced causal attention forward (K1).

    q: bf16 [q_rows, >= heads*d]; k_pool/v_pool: bf16 [pool_rows, >= kv_heads*d];
    chunk_rows: first pool row of every KV chunk (attention order).
    Returns (o bf16 [q_rows, heads*d], lse fp32 [heads, q_rows]).
    """
    assert q.dtype == torch.bfloat16 and k_pool.dtype == torch.bfloat16 and v_pool.dtype == torch.bfloat16
    if q.dim() == 3:  # [rows, heads, d] views
        head_dim = q.shape[-1]
        q, k_pool, v_pool = (x.reshape(x.shape[0], -1) for x in (q, k_pool, v_pool))
    assert q.is_cuda and q.stride(1) == 1 and k_pool.stride(1) == 1 and v_pool.stride(0) == k_pool.stride(0)
    q_rows = q.shape[0]
    d = head_dim or q.shape[1] // heads
    if o is None:
        o = torch.empty(q_rows, heads * d, dtype=torch.bfloat16, device=q.device)
    if lse is None:
        lse = torch.empty(heads, q_rows, dtype=torch.float32, device=q.device)
    rows, n = _rows(chunk_rows)
    N.check(N.lib().sp_attn_fwd(_ptr(q), q_rows, q.stride(0), _ptr(k_pool), _ptr(v_pool), k_pool.shape[0],
                                k_pool.stride(0), rows, n, chunk_len, heads, kv_heads, d, int(causal), _ptr(o),
                                o.stride(0), _ptr(lse), _stream()), "sp_attn_fwd")
    return o, lse


def attn_bwd(q, k_pool, v_pool, chunk_rows, chunk_len, heads, kv_heads, causal, o, lse, dout, dq_acc, dk_acc,
             dv_acc, acc_rows, delta_ws=None):
    """Backward of attn_fwd (K2): accumulates into fp32 dq_acc / dk_acc / dv_acc."""
    q_rows = q.shape[0]
    d = dq_acc.shape[1] // heads
    if delta_ws is None:
        delta_ws = torch.empty(2, heads, q_rows, dtype=torch.float32, device=q.device)
    rows, n = _rows(chunk_rows)
    arows, na = _rows(acc_rows)
    assert na == n
    N.check(N.lib().sp_attn_bwd(_ptr(q), q_rows, q.stride(0), _ptr(k_pool), _ptr(v_pool), k_pool.shape[0],
                                k_pool.stride(0), rows, n, chunk_len, heads, kv_heads, d, int(causal), _ptr(o),
                                o.stride(0), _ptr(dout), dout.stride(0), _ptr(lse), _ptr(delta_ws), _ptr(dq_acc),
                                _ptr(dk_acc), _ptr(dv_acc), dk_acc.shape[0], arows, _stream()), "sp_attn_bwd")
    return dq_acc, dk_acc, dv_acc


def attn_merge(o_a, lse_a, o_b, lse_b, heads, out=None, lse_out=None):
    """K3: merge two normalised partials (reference merge_partials + finalize)."""
    rows = o_a.shape[0]
    d = o_a.shape[1] // heads
    out = torch.empty_like(o_a) if out is None else out
    lse_out = torch.empty_like(lse_a) if lse_out is None else lse_out
    N.check(N.lib().sp_attn_merge(_ptr(o_a), _ptr(lse_a), _ptr(o_b), _ptr(lse_b), rows, heads, d, o_a.stride(0),
                                  _ptr(out), _ptr(lse_out), _stream()), "sp_attn_merge")
    return out, lse_out
