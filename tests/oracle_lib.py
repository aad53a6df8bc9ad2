"""Test-only loaders for the oracle libraries under oracle/_ref/.

  libpipelab_ref.so  the unmodified reference sources + oracle/ref_shim.cpp
                     (built only where /root/reference exists; travels to the
                     GPU box as a prebuilt file)
  liboracle.so       the C restatement oracle/attention_oracle.c (buildable
                     anywhere gcc is)
Nothing in the product imports this module.
"""
from __future__ import annotations

import ctypes as C
import json
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE = ROOT / "oracle"
REF_SO = ORACLE / "_ref" / "libpipelab_ref.so"
PORT_SO = ORACLE / "_ref" / "liboracle.so"
_ref = None
_port = None

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int)


def ref_available() -> bool:
    if REF_SO.exists():
        return True
    if Path("/root/reference/proj/src").exists():
        subprocess.run(["make", "-C", str(ORACLE), "ref"], check=True, capture_output=True)
        return REF_SO.exists()
    return False


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError("oracle/_ref/libpipelab_ref.so not built and /root/reference absent")
        _ref = C.CDLL(str(REF_SO))
        for fn in ["ref_schedule_json", "ref_validate_json", "ref_balance_json", "ref_exchange_json",
                   "ref_activation_json", "ref_exchange_volume", "ref_simulate_json", "ref_analytics_json", "ref_vocab_json", "ref_scenario_json",
                   "ref_gantt_json", "ref_gantt_measured"]:
            getattr(_ref, fn).restype = C.c_void_p
        _ref.ref_free.argtypes = [C.c_void_p]
        _ref.ref_schedule_json.argtypes = [C.c_int] * 5
        _ref.ref_validate_json.argtypes = [C.c_int] * 5
        _ref.ref_balance_json.argtypes = [C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.c_int, C.c_int]
        _ref.ref_exchange_json.argtypes = [C.c_int] * 5 + [C.c_double]
        _ref.ref_activation_json.argtypes = [C.POINTER(C.c_int64)] * 3 + [C.c_double]
        _ref.ref_exchange_volume.argtypes = [C.c_int64] * 5
        _ref.ref_analytics_json.argtypes = [C.c_int] + [C.c_int64] * 6
        _ref.ref_simulate_json.argtypes = [C.c_int] * 5 + [_dp, _dp, C.c_int64, C.POINTER(C.c_int64)]
        _ref.ref_vocab_json.argtypes = [C.c_int] * 5 + [C.c_double, C.c_double, C.c_int64]
        _ref.ref_scenario_json.argtypes = [C.c_char_p]
        _ref.ref_gantt_json.argtypes = [C.c_int] * 5 + [_dp, _dp, C.c_int64, C.c_int]
        _ref.ref_gantt_measured.argtypes = [C.c_int] * 4 + [C.POINTER(C.c_int32)] * 2 + [_dp, _dp, C.c_int]
        _ref.ref_chunk_attention.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, _ip, C.c_int, C.c_int, _dp, _dp,
                                             _dp, _dp]
        _ref.ref_merge.argtypes = [C.c_int, C.c_int] + [_dp] * 10
        _ref.ref_time_chunk_attention.restype = C.c_double
        _ref.ref_time_chunk_attention.argtypes = [C.c_int] * 5 + [C.c_ulonglong]
    return _ref


def ref_text(fn: str, *args) -> str:
    p = getattr(ref(), fn)(*args)
    try:
        return C.string_at(p).decode()
    finally:
        ref().ref_free(p)


def port():
    global _port
    if _port is None:
        if not PORT_SO.exists():
            subprocess.run(["make", "-C", str(ORACLE), "port"], check=True, capture_output=True)
        _port = C.CDLL(str(PORT_SO))
        _port.orc_chunk_attention.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_int, _ip, C.c_int,
                                              C.c_int, _dp, C.c_int, _dp, _dp, _dp]
        _port.orc_attn_bwd_head.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_int, C.c_int64,
                                            C.c_int, _dp, C.c_int, _dp, _dp, C.c_int, _dp, _dp, C.c_int]
        _port.orc_mha_fwd.argtypes = [_fp, C.c_int, C.c_int, C.c_int, _fp, _fp, C.c_int, _ip, C.c_int, C.c_int,
                                      _dp, _dp, C.c_int]
        _port.orc_mha_bwd.argtypes = [_fp, C.c_int, C.c_int, C.c_int, _fp, _fp, C.c_int, C.c_int64, C.c_int,
                                      _fp, _dp, _dp, _dp, _dp, C.c_int]
    return _port


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f(a: np.ndarray):
    return a.ctypes.data_as(_fp)


def ref_chunk_attention(q, k, v, chunk_sizes, causal):
    """Reference chunk_attention (one head, fp64).  Returns (out, partial, row_max, row_sumexp)."""
    q, k, v = (np.ascontiguousarray(x, dtype=np.float64) for x in (q, k, v))
    rows, d = q.shape
    out = np.zeros((rows, d))
    partial = np.zeros((rows, d))
    mx = np.zeros(rows)
    sm = np.zeros(rows)
    cs = (C.c_int * len(chunk_sizes))(*chunk_sizes)
    rc = ref().ref_chunk_attention(_d(q), rows, d, _d(k), _d(v), cs, len(chunk_sizes), int(causal), _d(out),
                                   _d(partial), _d(mx), _d(sm))
    assert rc == 0
    return out, partial, mx, sm


def port_chunk_attention(q, k, v, chunk_sizes, causal):
    """C restatement (one head, fp64).  Returns (out, lse, row_max, row_sumexp)."""
    q, k, v = (np.ascontiguousarray(x, dtype=np.float64) for x in (q, k, v))
    rows, d = q.shape
    out = np.zeros((rows, d))
    lse = np.zeros(rows)
    mx = np.zeros(rows)
    sm = np.zeros(rows)
    cs = (C.c_int * len(chunk_sizes))(*chunk_sizes)
    port().orc_chunk_attention(_d(q), d, rows, d, _d(k), _d(v), d, cs, len(chunk_sizes), int(causal), _d(out), d,
                               _d(lse), _d(mx), _d(sm))
    return out, lse, mx, sm


def port_attn_bwd_head(q, k, v, dout, lse, causal):
    q, k, v, dout, lse = (np.ascontiguousarray(x, dtype=np.float64) for x in (q, k, v, dout, lse))
    rows, d = q.shape
    total = k.shape[0]
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    port().orc_attn_bwd_head(_d(q), d, rows, d, _d(k), _d(v), d, total, int(causal), _d(dout), d, _d(lse), _d(dq),
                             d, _d(dk), _d(dv), d)
    return dq, dk, dv


def port_mha_fwd(q, k, v, chunk_sizes, causal, threads=8):
    """q [rows,a,d], k/v [total,g,d] float32 -> (o [rows,a,d] f64, lse [a,rows] f64)."""
    q, k, v = (np.ascontiguousarray(x, dtype=np.float32) for x in (q, k, v))
    rows, a, d = q.shape
    g = k.shape[1]
    o = np.zeros((rows, a, d))
    lse = np.zeros((a, rows))
    cs = (C.c_int * len(chunk_sizes))(*chunk_sizes)
    port().orc_mha_fwd(_f(q), rows, a, d, _f(k), _f(v), g, cs, len(chunk_sizes), int(causal), _d(o), _d(lse),
                       threads)
    return o, lse


def port_mha_bwd(q, k, v, dout, lse, causal, threads=8):
    q, k, v, dout = (np.ascontiguousarray(x, dtype=np.float32) for x in (q, k, v, dout))
    lse = np.ascontiguousarray(lse, dtype=np.float64)
    rows, a, d = q.shape
    total, g, _ = k.shape
    dq = np.zeros((rows, a, d))
    dk = np.zeros((total, g, d))
    dv = np.zeros((total, g, d))
    port().orc_mha_bwd(_f(q), rows, a, d, _f(k), _f(v), g, total, int(causal), _f(dout), _d(lse), _d(dq), _d(dk),
                       _d(dv), threads)
    return dq, dk, dv


def parse(text: str):
    return json.loads(text)


def _port_sampled():
    p = port()
    if not getattr(p, "_sampled_typed", False):
        p.orc_fwd_rows.argtypes = [_fp, C.c_int, C.c_int, C.c_int, _fp, _fp, C.c_int, C.c_int64, C.c_int, _ip,
                                   C.c_int, _dp, _dp, C.c_int]
        p.orc_bwd_rows.argtypes = [_fp, C.c_int, C.c_int, C.c_int, _fp, _fp, C.c_int, C.c_int64, C.c_int, _fp,
                                   C.c_int, _fp, C.c_int, _dp, _ip, C.c_int, _dp, C.c_int]
        p.orc_bwd_keys.argtypes = [_fp, C.c_int, C.c_int, C.c_int, _fp, _fp, C.c_int, C.c_int64, C.c_int, _fp,
                                   C.c_int, _fp, C.c_int, _dp, _ip, C.c_int, _dp, _dp, C.c_int]
        p._sampled_typed = True
    return p


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def port_fwd_rows(q, k, v, causal, sel, threads=8):
    """One head: q [rows,d], k/v [total,d] -> (o [len(sel),d], lse [len(sel)]) of rows `sel`."""
    q, k, v = _f32(q), _f32(k), _f32(v)
    rows, d = q.shape
    sel = np.ascontiguousarray(sel, dtype=np.int32)
    o = np.zeros((len(sel), d))
    lse = np.zeros(len(sel))
    _port_sampled().orc_fwd_rows(_f(q), d, rows, d, _f(k), _f(v), d, k.shape[0], int(causal),
                                 sel.ctypes.data_as(_ip), len(sel), _d(o), _d(lse), threads)
    return o, lse


def port_bwd_rows(q, k, v, o, dout, lse, causal, sel, threads=8):
    """dQ of rows `sel` for the backward as a function of (Q, K, V, O, dO, LSE)."""
    q, k, v, o, dout = _f32(q), _f32(k), _f32(v), _f32(o), _f32(dout)
    lse = np.ascontiguousarray(lse, dtype=np.float64)
    rows, d = q.shape
    sel = np.ascontiguousarray(sel, dtype=np.int32)
    dq = np.zeros((len(sel), d))
    _port_sampled().orc_bwd_rows(_f(q), d, rows, d, _f(k), _f(v), d, k.shape[0], int(causal), _f(o), d, _f(dout), d,
                                 _d(lse), sel.ctypes.data_as(_ip), len(sel), _d(dq), threads)
    return dq


def port_bwd_keys(q, k, v, o, dout, lse, causal, sel, threads=8):
    """dK/dV of key rows `sel`."""
    q, k, v, o, dout = _f32(q), _f32(k), _f32(v), _f32(o), _f32(dout)
    lse = np.ascontiguousarray(lse, dtype=np.float64)
    rows, d = q.shape
    sel = np.ascontiguousarray(sel, dtype=np.int32)
    dk = np.zeros((len(sel), d))
    dv = np.zeros((len(sel), d))
    _port_sampled().orc_bwd_keys(_f(q), d, rows, d, _f(k), _f(v), d, k.shape[0], int(causal), _f(o), d, _f(dout), d,
                                 _d(lse), sel.ctypes.data_as(_ip), len(sel), _d(dk), _d(dv), threads)
    return dk, dv
