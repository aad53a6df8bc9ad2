"""TEST INFRASTRUCTURE ONLY — float64 numpy oracle of one sliced-1F1B training
step of the Llama-style model the B200 executor trains (tiny config c1).

The reference (pipelab) has no model layers; SURVEY.md §8(c) asks for this
oracle to be new code whose attention is the reference's.  Attention forward
and backward go through oracle/attention_oracle.c (the C restatement of the
reference chunk_attention, attention.cpp:21-111, plus its exact backward),
here over the whole microbatch: slicing a causal sequence into n chunks and
attending slice i to chunks 1..i is exactly full causal attention (the point
of the reference's kernel tests, tests/test_attention.cpp:89-163), so the
step's loss and gradients must equal the unsliced computation.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
_lib = None
_lock = threading.Lock()
_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)


def lib():
    global _lib
    with _lock:
        if _lib is None:
            so = HERE / "_ref" / "liboracle.so"
            if not so.exists():
                subprocess.run(["make", "-C", str(HERE), "port"], check=True, capture_output=True)
            L = C.CDLL(str(so))
            L.orc_mha_fwd.argtypes = [_fp, C.c_int, C.c_int, C.c_int, _fp, _fp, C.c_int, C.POINTER(C.c_int), C.c_int,
                                      C.c_int, _dp, _dp, C.c_int]
            L.orc_mha_bwd.argtypes = [_fp, C.c_int, C.c_int, C.c_int, _fp, _fp, C.c_int, C.c_int64, C.c_int, _fp, _dp,
                                      _dp, _dp, _dp, C.c_int]
            _lib = L
    return _lib


THREADS = max(1, os.cpu_count() or 1)


def attn_fwd(q, k, v, chunk_len):
    """q [S,a,d], k/v [S,g,d] -> (o [S,a,d], lse [a,S]); causal over chunks of chunk_len."""
    S, a, d = q.shape
    g = k.shape[1]
    qf, kf, vf = (np.ascontiguousarray(x, dtype=np.float32) for x in (q, k, v))
    o = np.zeros((S, a, d))
    lse = np.zeros((a, S))
    n = S // chunk_len
    cs = (C.c_int * n)(*([chunk_len] * n))
    lib().orc_mha_fwd(qf.ctypes.data_as(_fp), S, a, d, kf.ctypes.data_as(_fp), vf.ctypes.data_as(_fp), g, cs, n, 1,
                      o.ctypes.data_as(_dp), lse.ctypes.data_as(_dp), THREADS)
    return o, lse


def attn_bwd(q, k, v, do, lse):
    S, a, d = q.shape
    g = k.shape[1]
    qf, kf, vf, dof = (np.ascontiguousarray(x, dtype=np.float32) for x in (q, k, v, do))
    lse = np.ascontiguousarray(lse, dtype=np.float64)
    dq = np.zeros((S, a, d))
    dk = np.zeros((S, g, d))
    dv = np.zeros((S, g, d))
    lib().orc_mha_bwd(qf.ctypes.data_as(_fp), S, a, d, kf.ctypes.data_as(_fp), vf.ctypes.data_as(_fp), g, S, 1,
                      dof.ctypes.data_as(_fp), lse.ctypes.data_as(_dp), dq.ctypes.data_as(_dp),
                      dk.ctypes.data_as(_dp), dv.ctypes.data_as(_dp), THREADS)
    return dq, dk, dv


def rope_tables(S, d, theta):
    j = np.arange(d // 2, dtype=np.float64)
    inv = theta ** (-2.0 * j / d)
    ang = np.arange(S, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang), np.sin(ang)


def rope(x, cos, sin):  # x [S, heads, d], rotate-half pairs (j, j+d/2)
    h = x.shape[-1] // 2
    x1, x2 = x[..., :h], x[..., h:]
    c, s = cos[:, None, :], sin[:, None, :]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def rope_bwd(g, cos, sin):
    h = g.shape[-1] // 2
    g1, g2 = g[..., :h], g[..., h:]
    c, s = cos[:, None, :], sin[:, None, :]
    return np.concatenate([g1 * c + g2 * s, g2 * c - g1 * s], axis=-1)


def rmsnorm(x, w, eps):
    r = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    return x * r * w, r


def rmsnorm_bwd(dy, x, w, r):
    g = dy * w
    dim = x.shape[-1]
    dx = r * (g - x * (r * r) * np.sum(g * x, axis=-1, keepdims=True) / dim)
    dw = np.sum(dy * x * r, axis=0)
    return dx, dw


def silu(x):
    return x / (1.0 + np.exp(-x))


class Model:
    """Weights: dict with per-layer lists 'attn_norm','wqkv','wo','mlp_norm','wgu','wd'
    and 'embedding','final_norm','head' (float64 arrays, row-major like the GPU)."""

    def __init__(self, weights, heads, kv_heads, rope_theta=10000.0, eps=1e-5):
        self.w = weights
        self.a = heads
        self.g = kv_heads
        self.theta = rope_theta
        self.eps = eps

    def step(self, tokens, targets, slices):
        """Mean loss over all microbatches and the gradients (same structure as weights)."""
        W = self.w
        L = len(W["wqkv"])
        grads = {k: ([np.zeros_like(x) for x in v] if isinstance(v, list) else np.zeros_like(v)) for k, v in W.items()}
        m, S = tokens.shape
        total = float(np.sum(targets >= 0))
        loss = 0.0
        h = W["embedding"].shape[1]
        d = h // self.a
        H = W["wd"][0].shape[1]
        cos, sin = rope_tables(S, d, self.theta)
        for b in range(m):
            x = W["embedding"][tokens[b]].astype(np.float64)
            cache = []
            for l in range(L):
                xn, r1 = rmsnorm(x, W["attn_norm"][l], self.eps)
                qkv = xn @ W["wqkv"][l].T
                q = rope(qkv[:, :self.a * d].reshape(S, self.a, d), cos, sin)
                k = rope(qkv[:, self.a * d:(self.a + self.g) * d].reshape(S, self.g, d), cos, sin)
                v = qkv[:, (self.a + self.g) * d:].reshape(S, self.g, d)
                o, lse = attn_fwd(q, k, v, S // slices)
                o2 = o.reshape(S, self.a * d)
                x_mid = x + o2 @ W["wo"][l].T
                xn2, r2 = rmsnorm(x_mid, W["mlp_norm"][l], self.eps)
                gu = xn2 @ W["wgu"][l].T
                gate, up = gu[:, :H], gu[:, H:]
                act = silu(gate) * up
                x_out = x_mid + act @ W["wd"][l].T
                cache.append((x, xn, r1, q, k, v, o, o2, lse, x_mid, xn2, r2, gate, up, act))
                x = x_out
            xf, rf = rmsnorm(x, W["final_norm"], self.eps)
            logits = xf @ W["head"].T
            mx = logits.max(axis=1, keepdims=True)
            p = np.exp(logits - mx)
            se = p.sum(axis=1, keepdims=True)
            lse_l = (mx + np.log(se))[:, 0]
            valid = targets[b] >= 0
            idx = np.where(valid, targets[b], 0)
            loss += float(np.sum((lse_l - logits[np.arange(S), idx])[valid]))
            dlog = p / se
            dlog[np.arange(S), idx] -= 1.0
            dlog[~valid] = 0.0
            dlog /= total
            grads["head"] += dlog.T @ xf
            dxf = dlog @ W["head"]
            dx, dw = rmsnorm_bwd(dxf, x, W["final_norm"], rf)
            grads["final_norm"] += dw
            for l in reversed(range(L)):
                (x_in, xn, r1, q, k, v, o, o2, lse, x_mid, xn2, r2, gate, up, act) = cache[l]
                # MLP
                grads["wd"][l] += dx.T @ act
                dact = dx @ W["wd"][l]
                sg = 1.0 / (1.0 + np.exp(-gate))
                dgate = dact * up * (sg * (1.0 + gate * (1.0 - sg)))
                dup = dact * gate * sg
                dgu = np.concatenate([dgate, dup], axis=1)
                grads["wgu"][l] += dgu.T @ xn2
                dxn2 = dgu @ W["wgu"][l]
                dxm, dw = rmsnorm_bwd(dxn2, x_mid, W["mlp_norm"][l], r2)
                grads["mlp_norm"][l] += dw
                dx = dx + dxm
                # attention
                grads["wo"][l] += dx.T @ o2
                do = (dx @ W["wo"][l]).reshape(S, self.a, d)
                dq, dk, dv = attn_bwd(q, k, v, do, lse)
                dq = rope_bwd(dq, cos, sin)
                dk = rope_bwd(dk, cos, sin)
                dqkv = np.concatenate([dq.reshape(S, -1), dk.reshape(S, -1), dv.reshape(S, -1)], axis=1)
                grads["wqkv"][l] += dqkv.T @ xn
                dxn = dqkv @ W["wqkv"][l]
                dxa, dw = rmsnorm_bwd(dxn, x_in, W["attn_norm"][l], r1)
                grads["attn_norm"][l] += dw
                dx = dx + dxa
            np.add.at(grads["embedding"], tokens[b], dx)
        return loss / total, grads


def time_step(model: Model, tokens, targets, slices):
    t0 = time.perf_counter()
    loss, _ = model.step(tokens, targets, slices)
    return time.perf_counter() - t0, loss
