"""The C-ABI library builds, loads without a GPU and exports every symbol that
include/slimpipe.h declares (no compute calls here)."""
import ctypes
import re

import pytest
from pathlib import Path

from paper_2504_14519_b200 import native

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "slimpipe.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sp_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    lib = native.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_status_strings_and_errors_without_gpu():
    lib = native.lib()
    assert lib.sp_status_string(0) == b"ok"
    assert lib.sp_version() >= 1
    # invalid shapes are rejected before touching the device
    rows = (ctypes.c_int32 * 1)(0)
    rc = lib.sp_attn_fwd(None, 100, 128, None, None, 128, 128, rows, 1, 128, 1, 1, 128, 1, None, 128, None, None)
    assert rc == native.SP_ERR_UNSUPPORTED
    assert b"multiples of 128" in lib.sp_last_error()


@pytest.mark.parametrize("kw,msg", [
    ({"layers": 3, "pp": 2}, b"must divide by pp"),
    ({"slices": 3}, b"divisible by slices"),
    ({"pp": 2, "slices": 3, "seq_len": 3072, "layers": 2}, b"multiple of p"),   # schedule.cpp:249-252
    ({"pp": 2, "microbatches": 0, "layers": 2}, b"m must be >= 1"),
    ({"hidden": 250}, b"heads * head_dim"),
])
def test_runtime_rejects_invalid_configs_before_touching_the_device(kw, msg):
    """Reference error behaviour (std::invalid_argument <-> SP_ERR_INVALID),
    checked host-side before any CUDA call, so it runs without a GPU."""
    from paper_2504_14519_b200.runtime import StepConfig, _lib
    lib = _lib()
    c = StepConfig.c1(**kw).to_c(0)
    h = ctypes.c_void_p()
    assert lib.sp_runtime_create(ctypes.byref(c), None, ctypes.byref(h)) == native.SP_ERR_INVALID
    assert msg in lib.sp_last_error()
    c = StepConfig.c1().to_c(0)
    c.recompute = 7
    assert lib.sp_runtime_create(ctypes.byref(c), None, ctypes.byref(h)) == native.SP_ERR_INVALID


@pytest.mark.parametrize("kw,code,msg", [
    ({"pp": 3, "layers": 6, "slices": 3, "seq_len": 3072, "interleave": 2}, "SP_ERR_UNSUPPORTED", b"even pp"),
    ({"pp": 2, "layers": 4, "interleave": 2, "vocab_parallel": True}, "SP_ERR_UNSUPPORTED", b"vocab_parallel 0"),
    ({"pp": 2, "layers": 4, "interleave": 2, "exchange": "on"}, "SP_ERR_UNSUPPORTED", b"exchange off"),
    ({"pp": 2, "layers": 6, "interleave": 2}, "SP_ERR_INVALID", b"pp*v"),
    ({"pp": 2, "layers": 2, "vocab": 1002, "vocab_parallel": True}, "SP_ERR_INVALID", b"multiple of 4"),
    ({"slices": 512, "seq_len": 512 * 128}, "SP_ERR_UNSUPPORTED", b"SP_MAX_CHUNKS"),  # before any NCCL call
    ({"pp": 2, "layers": 4, "vocab": 1024, "vocab_parallel": True, "exchange": "on"}, "SP_ERR_UNSUPPORTED",
     b"exchange off"),
    ({"pp": 2, "layers": 4, "exchange": "on", "exchange_min_chunks": -1}, "SP_ERR_INVALID", b"exchange_min_chunks"),
    ({"pp": 2, "layers": 4, "exchange": "on", "exchange_skip_last": 2}, "SP_ERR_INVALID", b"exchange_skip_last"),
])
def test_experimental_paths_reject_unsupported_configs_host_side(kw, code, msg):
    """Interleaving / vocabulary parallelism preconditions (runtime.cpp init),
    checked before any CUDA or NCCL call."""
    from paper_2504_14519_b200.runtime import StepConfig, _lib
    lib = _lib()
    c = StepConfig.c1(**kw).to_c(0)
    h = ctypes.c_void_p()
    assert lib.sp_runtime_create(ctypes.byref(c), None, ctypes.byref(h)) == getattr(native, code)
    assert msg in lib.sp_last_error()
