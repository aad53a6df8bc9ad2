"""Python host mirror of the step executor (csrc/host/runtime.cpp) — the
call a user makes to run SlimPipe sliced-1F1B training steps on B200s.

    cfg = StepConfig.c2(layers=8)             # Llama-7B layer shapes, 128K ctx
    step = SlimPipeStep(cfg)                  # rank/world from torchrun env
    loss = step.step(tokens, targets)         # one optimizer step

Process model: one process per GPU (torchrun); rank r runs stage r+1; the
NCCL communicators of the executor are bootstrapped through
torch.distributed (plumbing only).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, replace

import numpy as np

from . import native as N


class _Cfg(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("layers", "hidden", "ffn_hidden", "heads", "kv_heads", "head_dim", "vocab",
                                         "microbatches", "slices", "pp", "rank", "exchange_mode")] + [
        ("seq_len", C.c_int64), ("rope_theta", C.c_float), ("norm_eps", C.c_float), ("lr", C.c_float),
        ("seed", C.c_uint64), ("recompute", C.c_int32), ("vocab_parallel", C.c_int32),
        ("interleave", C.c_int32), ("offload", C.c_int32), ("dkv_bf16", C.c_int32),
        ("exchange_min_chunks", C.c_int32), ("exchange_skip_last", C.c_int32)]


RECOMPUTE = {"selective": 0, "full": 1, "auto": 2}


@dataclass(frozen=True)
class StepConfig:
    layers: int
    hidden: int
    ffn_hidden: int
    heads: int
    kv_heads: int
    vocab: int
    seq_len: int
    slices: int
    microbatches: int
    pp: int = 1
    exchange: str = "off"
    recompute: str = "auto"  # "selective": stash attention O/LSE, "full": K1 again in the backward, "auto": selective if it fits
    vocab_parallel: bool = False  # LM head + cross entropy split by vocabulary across the pp stages
    interleave: int = 1  # v stages per device (interleaved SlimPipe; even pp, exchange off)
    offload: bool = False  # stage inputs + attention O/LSE to pinned host memory between F and BW
    dkv_bf16: bool = False  # dK/dV chunk accumulators stored in bf16 (half their HBM)
    exchange_min_chunks: int = 0  # exchange placement: drop plan transfers moving fewer KV chunks
    exchange_skip_last: bool = False  # exchange placement: drop plan transfers into the last stage
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5
    lr: float = 1e-4
    seed: int = 1234

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    @property
    def slice_len(self) -> int:
        return self.seq_len // self.slices

    # BASELINE.json configs
    @staticmethod
    def c1(**kw) -> "StepConfig":
        """tiny Llama-style: 4 layers, h256, 4 heads (d64), 4K seq, 4 slices, m2."""
        return replace(StepConfig(4, 256, 1024, 4, 4, 1000, 4096, 4, 2), **kw)

    @staticmethod
    def c2(**kw) -> "StepConfig":
        """Llama-7B layer shapes, 128K context, 8 slices, m4 (depth reduced)."""
        return replace(StepConfig(8, 4096, 11008, 32, 32, 32000, 131072, 8, 4), **kw)

    @staticmethod
    def c3(**kw) -> "StepConfig":
        """Llama-13B layer shapes, 256K context, 16 slices, m4."""
        return replace(StepConfig(40, 5120, 13824, 40, 40, 128000, 262144, 16, 4), **kw)

    @staticmethod
    def c4(**kw) -> "StepConfig":
        """Llama-70B layer shapes (GQA 64/8), 1M context, 32 slices, m1 (depth reduced)."""
        return replace(StepConfig(16, 8192, 28672, 64, 8, 128000, 1 << 20, 32, 1), **kw)

    @staticmethod
    def from_scenario(text: str, **overrides) -> "StepConfig":
        """A reference scenario file (scenario.cpp schema) as the executed step:
        the same file drives plan.simulate / plan.gantt_text and the GPU run.
        Only what the executor runs is accepted: scheme slimpipe, tp = cp = dp
        = ep = 1, checkpointing selective or full."""
        from . import plan as P
        sc = P.scenario(text)  # strict: unknown fields and bad values raise ValueError
        md, pa, rn = sc["model"], sc["parallelism"], sc["run"]
        if sc["scheme"] != "slimpipe":
            raise ValueError(f"scenario: the executor runs scheme slimpipe, not {sc['scheme']}")
        for k in ("tp", "cp", "dp", "ep"):
            if pa[k] != 1:
                raise ValueError(f"scenario: {k} = {pa[k]} is not on the executed path (pipeline only)")
        if rn["checkpointing"] not in ("selective", "full"):
            raise ValueError(f"scenario: checkpointing {rn['checkpointing']} (the executor recomputes: selective|full)")
        # offload_ratio > 0 runs the executor's activation offload, which moves
        # every activation but the K/V chunks (stage inputs, attention O/LSE)
        # to the host — the ratio itself is not tunable
        kw = dict(layers=md["layers"], hidden=md["hidden"], ffn_hidden=md["ffn"], heads=md["heads"],
                  kv_heads=md["query_groups"], vocab=md["vocab"], seq_len=rn["seq_len"], slices=rn["slices"],
                  microbatches=rn["microbatches"], pp=pa["pp"], interleave=pa["stages_per_device"],
                  exchange=sc["exchange"], recompute=rn["checkpointing"], vocab_parallel=bool(rn["vocab_parallel"]),
                  offload=rn["offload_ratio"] > 0, seed=sc["seed"])
        kw.update(overrides)
        return StepConfig(**kw)

    def to_c(self, rank: int) -> _Cfg:
        return _Cfg(self.layers, self.hidden, self.ffn_hidden, self.heads, self.kv_heads, self.head_dim, self.vocab,
                    self.microbatches, self.slices, self.pp, rank, N.MODES[self.exchange], self.seq_len,
                    self.rope_theta, self.norm_eps, self.lr, self.seed, RECOMPUTE[self.recompute],
                    int(self.vocab_parallel), int(self.interleave), int(self.offload), int(self.dkv_bf16),
                    int(self.exchange_min_chunks), int(self.exchange_skip_last))

    # ---- accounting ----
    def linear_params_per_layer(self) -> int:
        h, H, kvd = self.hidden, self.ffn_hidden, self.kv_heads * self.head_dim
        return 2 * h * h + 2 * h * kvd + 3 * h * H

    def model_flops_per_step(self) -> float:
        """F_model = 3 (2 N_lin + 2 h V) m S + 3 m L 2 h S (S+1)  (fwd+bwd, causal
        attention counted once per pair, no recompute)."""
        m, S, L, h = self.microbatches, self.seq_len, self.layers, self.hidden
        n_lin = L * self.linear_params_per_layer()
        return 3.0 * (2 * n_lin + 2 * h * self.vocab) * m * S + 3.0 * m * L * 2 * h * S * (S + 1)


_PARAM_NAMES = ["attn_norm", "wqkv", "wo", "mlp_norm", "wgu", "wd", "embedding", "final_norm", "head"]


def _lib():
    lib = N.lib()
    lib.sp_nccl_unique_id.argtypes = [C.c_void_p]
    lib.sp_runtime_create.argtypes = [C.POINTER(_Cfg), C.c_void_p, C.POINTER(C.c_void_p)]
    lib.sp_runtime_create_loopback.argtypes = [C.POINTER(_Cfg), C.c_void_p, C.POINTER(C.c_void_p)]
    lib.sp_loopback_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
    lib.sp_loopback_destroy.argtypes = [C.c_void_p]
    lib.sp_loopback_errors.argtypes = [C.c_void_p]
    lib.sp_loopback_pingpong.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int]
    lib.sp_loopback_pingpong_1thread.argtypes = [C.c_void_p] + [C.c_void_p] * 4 + [C.c_int64, C.c_int]
    lib.sp_runtime_exchange_stats.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
    lib.sp_runtime_comm_stats.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
    lib.sp_runtime_enqueue_position.argtypes = [C.c_void_p]
    lib.sp_runtime_destroy.argtypes = [C.c_void_p]
    lib.sp_runtime_step.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_float)]
    lib.sp_runtime_sync.argtypes = [C.c_void_p]
    lib.sp_runtime_stream.argtypes = [C.c_void_p]
    lib.sp_runtime_stream.restype = C.c_void_p
    lib.sp_runtime_timeline.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int]
    lib.sp_runtime_attn_stats.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
    lib.sp_runtime_memory.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
    lib.sp_runtime_recompute.argtypes = [C.c_void_p]
    lib.sp_runtime_offload_bytes.argtypes = [C.c_void_p]
    lib.sp_runtime_offload_bytes.restype = C.c_longlong
    lib.sp_runtime_progress.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]
    lib.sp_runtime_param.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_int]
    return lib


N_NCCL_IDS = 4  # stage fwd, stage bwd, fwd-tick exchange, bwd-tick exchange


def make_nccl_ids() -> bytes:
    out = b""
    for _ in range(N_NCCL_IDS):
        buf = C.create_string_buffer(128)
        N.check(_lib().sp_nccl_unique_id(buf), "sp_nccl_unique_id")
        out += buf.raw
    return out


def nccl_ids(rank: int, world: int):
    """The executor's NCCL unique ids, made on rank 0 and broadcast with
    torch.distributed (which must be initialised when world > 1)."""
    if world == 1:
        return None
    import torch.distributed as dist
    ids = [make_nccl_ids() if rank == 0 else None]
    dist.broadcast_object_list(ids, src=0)
    return C.create_string_buffer(ids[0], 128 * N_NCCL_IDS)


class LoopbackWorld:
    """All pp ranks of a step as threads of this process on ONE GPU
    (csrc/host/transport.hpp loopback): the stage links and exchange
    transfers run through device flags and copy kernels instead of NCCL,
    with the executor's own send/recv program.  For single-GPU boxes/tests:

        world = LoopbackWorld(cfg.pp)
        steps = [SlimPipeStep(cfg, r, cfg.pp, loopback=world) for r in range(cfg.pp)]
        losses = world.run(lambda r: steps[r].step(tok, tgt, optimizer=False))
    """

    def __init__(self, ranks: int):
        self.ranks = ranks
        h = C.c_void_p()
        N.check(_lib().sp_loopback_create(ranks, C.byref(h)), "sp_loopback_create")
        self._h = h

    @property
    def handle(self):
        return self._h

    def errors(self) -> int:
        return int(_lib().sp_loopback_errors(self._h))

    def run(self, fn, timeout: float | None = None, steps=None):
        """fn(rank) on one host thread per rank (concurrently, as the ranks'
        enqueues must be); returns the per-rank results, re-raising the
        first exception.  With `timeout` (seconds) a stuck step raises
        TimeoutError naming, per rank of `steps`, the pass the host is
        enqueuing and the first pass not finished on the device."""
        import threading
        import time
        out, err = [None] * self.ranks, [None] * self.ranks

        def body(r):
            try:
                out[r] = fn(r)
            except BaseException as e:  # noqa: BLE001 - re-raised below
                err[r] = e
        ths = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(self.ranks)]
        for t in ths:
            t.start()
        t_end = None if timeout is None else time.monotonic() + timeout
        for t in ths:
            t.join(None if t_end is None else max(0.0, t_end - time.monotonic()))
        if any(t.is_alive() for t in ths):
            where = [] if steps is None else [
                f"rank {r}: host enqueuing pass #{_lib().sp_runtime_enqueue_position(s._h)}, device at {s.progress()}"
                for r, s in enumerate(steps)]
            # the device is wedged: no cleanup can complete (stream syncs would
            # block forever), so report and end the process
            import sys
            print(f"loopback step did not finish in {timeout} s; " + "; ".join(where), file=sys.stderr, flush=True)
            os._exit(3)
        for e in err:
            if e is not None:
                raise e
        return out

    def close(self):
        if getattr(self, "_h", None):
            _lib().sp_loopback_destroy(self._h)
            self._h = None


class SlimPipeStep:
    """One pipeline stage of the sliced-1F1B step on this process's GPU."""

    def __init__(self, cfg: StepConfig, rank: int | None = None, world: int | None = None,
                 loopback: LoopbackWorld | None = None):
        self.cfg = cfg
        self.rank = int(os.environ.get("RANK", 0)) if rank is None else rank
        self.world = int(os.environ.get("WORLD_SIZE", 1)) if world is None else world
        if cfg.pp != self.world:
            raise ValueError(f"pp ({cfg.pp}) must equal the number of ranks ({self.world})")
        lib = _lib()
        h = C.c_void_p()
        c = cfg.to_c(self.rank)
        if loopback is not None:
            N.check(lib.sp_runtime_create_loopback(C.byref(c), loopback.handle, C.byref(h)),
                    "sp_runtime_create_loopback")
        else:
            ids = nccl_ids(self.rank, self.world)
            N.check(lib.sp_runtime_create(C.byref(c), ids, C.byref(h)), "sp_runtime_create")
        self._h = h
        self.stage = self.rank + 1
        self.is_first = self.stage == 1
        self.is_last = self.stage == cfg.pp

    def global_layer(self, local: int) -> int:
        """Model layer index of this device's local layer `local` (= c*Lps + l:
        layer l of stage rank+1+c*pp)."""
        c = self.cfg
        lps = c.layers // (c.pp * c.interleave)
        return ((local // lps) * c.pp + self.rank) * lps + local % lps

    def close(self):
        if getattr(self, "_h", None):
            _lib().sp_runtime_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream_handle(self) -> int:
        return _lib().sp_runtime_stream(self._h)

    def step(self, tokens, targets, optimizer: bool = True, on_device: bool = False) -> float:
        """Run all passes of this stage's program for m microbatches.

        tokens/targets: int32 [microbatches, seq_len] — numpy (host) arrays, or
        device pointers (ints) when on_device.  Returns the mean loss on the
        last stage (0.0 elsewhere).
        """
        loss = C.c_float(0.0)
        if on_device:
            tp, gp = C.c_void_p(tokens), C.c_void_p(targets)
        else:
            tokens = np.ascontiguousarray(tokens, dtype=np.int32)
            targets = np.ascontiguousarray(targets, dtype=np.int32)
            tp, gp = tokens.ctypes.data_as(C.c_void_p), targets.ctypes.data_as(C.c_void_p)
        flags = 0 if optimizer else 1
        N.check(_lib().sp_runtime_step(self._h, tp, gp, int(on_device), flags, C.byref(loss)), "sp_runtime_step")
        return float(loss.value)

    def step_async(self, tokens_dev: int, targets_dev: int, optimizer: bool = True) -> None:
        """Enqueue one step with device-resident inputs; no host synchronisation."""
        N.check(_lib().sp_runtime_step(self._h, C.c_void_p(tokens_dev), C.c_void_p(targets_dev), 1,
                                       0 if optimizer else 1, None), "sp_runtime_step")

    def progress(self):
        """(position, (kind, microbatch, slice, stage)) of the first unfinished
        pass of the last enqueued step on the compute stream, or None."""
        b = (C.c_int32 * 4)()
        x = _lib().sp_runtime_progress(self._h, b)
        return None if x < 0 else (x, tuple(b))

    def sync(self):
        N.check(_lib().sp_runtime_sync(self._h), "sp_runtime_sync")

    def timeline(self):
        c = self.cfg
        vp = c.vocab_parallel and c.pp > 1  # + one VocabForward and one VocabBackward per slice
        n_pass = (4 if vp else 2) * c.interleave * c.microbatches * c.slices
        buf = (C.c_double * (1 + 3 * n_pass))()
        n = _lib().sp_runtime_timeline(self._h, buf, len(buf))
        if n < 0:
            N.check(n, "sp_runtime_timeline")
        vals = list(buf[:n])
        return vals[0], [(int(vals[i]), vals[i + 1], vals[i + 2]) for i in range(1, n, 3)]

    def attn_stats(self) -> dict:
        b = (C.c_double * 6)()
        N.check(_lib().sp_runtime_attn_stats(self._h, b), "sp_runtime_attn_stats")
        return {"fwd_ms": b[0], "fwd_flops": b[1], "fwd_launches": int(b[2]), "bwd_ms": b[3], "bwd_flops": b[4],
                "bwd_launches": int(b[5])}

    def memory(self) -> dict:
        b = (C.c_int64 * 7)()
        N.check(_lib().sp_runtime_memory(self._h, b), "sp_runtime_memory")
        keys = ["slots", "slots_high_water", "slot_bytes", "ledger_peak_units", "bytes_allocated", "n_params",
                "layers_per_stage"]
        out = dict(zip(keys, list(b)))
        out["recompute"] = "full" if _lib().sp_runtime_recompute(self._h) else "selective"
        out["offload_host_bytes"] = int(_lib().sp_runtime_offload_bytes(self._h))
        return out

    def exchange_stats(self) -> dict:
        b = (C.c_int64 * 3)()
        N.check(_lib().sp_runtime_exchange_stats(self._h, b), "sp_runtime_exchange_stats")
        return {"passes_out": b[0], "passes_in": b[1], "bytes_sent": b[2]}

    def comm_stats(self) -> dict:
        """Stage sends of the last step (CUDA events on the send streams)."""
        b = (C.c_double * 4)()
        N.check(_lib().sp_runtime_comm_stats(self._h, b), "sp_runtime_comm_stats")
        return {"messages": int(b[0]), "bytes": b[1], "send_ms": b[2], "fastest_ms": b[3]}

    # ---- parameter access (tests) ----
    def _param_shape(self, which: str):
        c = self.cfg
        h, H, qkv = c.hidden, c.ffn_hidden, (c.heads + 2 * c.kv_heads) * c.head_dim
        return {"attn_norm": (h,), "wqkv": (qkv, h), "wo": (h, c.heads * c.head_dim), "mlp_norm": (h,),
                "wgu": (2 * H, h), "wd": (h, H), "embedding": (c.vocab, h), "final_norm": (h,),
                "head": (c.vocab // c.pp if (c.vocab_parallel and c.pp > 1) else c.vocab, h)}[which]

    def _param_io(self, layer: int, which: str, arr: np.ndarray | None, direction: int) -> np.ndarray:
        shape = self._param_shape(which)
        if arr is None:
            arr = np.zeros(shape, np.float32)
        arr = np.ascontiguousarray(arr, dtype=np.float32)
        assert arr.shape == shape
        N.check(_lib().sp_runtime_param(self._h, layer, _PARAM_NAMES.index(which), arr.ctypes.data_as(C.c_void_p),
                                        arr.size, direction), "sp_runtime_param")
        return arr

    def get_param(self, layer: int, which: str) -> np.ndarray:
        return self._param_io(layer, which, None, 0)

    def set_param(self, layer: int, which: str, value: np.ndarray) -> None:
        self._param_io(layer, which, value, 1)

    def get_grad(self, layer: int, which: str) -> np.ndarray:
        return self._param_io(layer, which, None, 2)
