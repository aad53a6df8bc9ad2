"""ctypes binding of libslimpipe.so (the C-ABI in include/slimpipe.h).

This is plumbing: it loads the in-tree library, declares argument types and
turns status codes into exceptions with the reference's error classes
(std::invalid_argument -> ValueError, std::runtime_error -> RuntimeError).
There is deliberately no fallback: if the library is missing or fails to
load, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["SP_LIB"]) if os.environ.get("SP_LIB") else _PKG / "lib" / "libslimpipe.so"  # SP_LIB: A/B builds
_lib: C.CDLL | None = None

SP_OK, SP_ERR_INVALID, SP_ERR_RUNTIME, SP_ERR_CUDA, SP_ERR_NCCL, SP_ERR_UNSUPPORTED, SP_ERR_NO_DEVICE = range(7)

SCHEMES = {"gpipe": 0, "terapipe": 1, "1f1b": 2, "interleaved_1f1b": 3, "zbv": 4, "vhalf": 5, "slimpipe": 6}
MODES = {"off": 0, "on": 1, "early": 2}

_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_f64p = C.POINTER(C.c_double)
_charpp = C.POINTER(C.c_void_p)

# name -> (restype, argtypes)
_SIGS = {
    "sp_status_string": (C.c_char_p, [C.c_int]),
    "sp_last_error": (C.c_char_p, []),
    "sp_free": (None, [C.c_void_p]),
    "sp_version": (C.c_int, []),
    "sp_launch_count": (C.c_longlong, []),
    "sp_library_launch_count": (C.c_longlong, []),
    "sp_gemm_plans_json": (C.c_int, [_charpp]),
    "sp_plan_schedule_json": (C.c_int, [C.c_int] * 5 + [_charpp]),
    "sp_plan_validate_json": (C.c_int, [C.c_int] * 5 + [_charpp]),
    "sp_plan_balance_json": (C.c_int, [_i64p, _i32p, C.c_int, C.c_int, _charpp]),
    "sp_plan_exchange_json": (C.c_int, [C.c_int] * 5 + [C.c_double, _charpp]),
    "sp_exchange_passes_json": (C.c_int, [C.c_int] * 7 + [_charpp]),
    "sp_plan_activation_json": (C.c_int, [_i64p, _i64p, _i64p, C.c_double, _charpp]),
    "sp_plan_exchange_volume": (C.c_int, [C.c_int64] * 5 + [_charpp]),
    "sp_plan_analytics_json": (C.c_int, [C.c_int] + [C.c_int64] * 6 + [_charpp]),
    "sp_plan_simulate_json": (C.c_int, [C.c_int] * 5 + [_f64p, _f64p, C.c_int64, _i64p, _charpp]),
    "sp_plan_vocab_json": (C.c_int, [C.c_int] * 5 + [C.c_double, C.c_double, C.c_int64, _charpp]),
    "sp_plan_scenario_json": (C.c_int, [C.c_char_p, _charpp]),
    "sp_plan_gantt_json": (C.c_int, [C.c_int] * 5 + [_f64p, _f64p, C.c_int64, C.c_int, _charpp]),
    "sp_plan_gantt_measured": (C.c_int, [C.c_int] * 5 + [C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                                         _f64p, _f64p, C.c_int, _charpp]),
    "sp_plan_metrics_measured": (C.c_int, [C.c_int] * 5 + [C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                                           _f64p, _f64p, _charpp]),
    "sp_attn_fwd": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                              _i32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                              C.c_int64, C.c_void_p, C.c_void_p]),
    "sp_attn_bwd": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                              _i32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                              C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_int64, _i32p, C.c_void_p]),
    "sp_attn_merge": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int,
                                C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
}


def lib() -> C.CDLL:
    """Load (once) and type the in-tree libslimpipe.so; raise if absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is not built; run `python -m paper_2504_14519_b200.build` "
                               "(there is no fallback implementation)")
        # torch first: the library links NCCL by soname, and the process must
        # hold torch's (newer) libnccl.so.2 — loaded after an older system copy,
        # libtorch_cuda fails on symbols the older one lacks
        import torch  # noqa: F401
        handle = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name, None)
            if fn is None:
                continue  # checked by tests/test_abi.py against include/slimpipe.h
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(code: int, what: str = "") -> None:
    if code == SP_OK:
        return
    msg = (lib().sp_last_error() or b"").decode() or lib().sp_status_string(code).decode()
    if code == SP_ERR_INVALID:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: [{lib().sp_status_string(code).decode()}] {msg}")


def _json_call(fn_name: str, *args):
    out = C.c_void_p()
    code = getattr(lib(), fn_name)(*args, C.byref(out))
    try:
        text = C.string_at(out.value).decode() if out.value else ""
    finally:
        if out.value:
            lib().sp_free(out)
    if code != SP_OK:
        err = json.loads(text) if text.startswith("{") else {}
        cls = ValueError if code == SP_ERR_INVALID else RuntimeError
        raise cls(err.get("what", text))
    return text


def arr(ctype, values):
    values = list(values)
    return (ctype * max(1, len(values)))(*values)
