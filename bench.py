#!/usr/bin/env python
"""SlimPipe sliced-1F1B training step on B200 — benchmark (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

Workload (BASELINE.json configs[1]): Llama-7B layer shapes
(h 4096, 32 heads x d128, FFN 11008, V 32000), depth reduced to --layers
(default 8), 128K-token microbatches cut into 8 slices of 16K, m=4
microbatches, pipeline PP = N GPUs (layers/N per stage), synthetic tokens,
random-init weights, bf16 compute with fp32 accumulation/master weights,
AdamW step included.  Total work per step is fixed as N grows ("strong").

value      tokens/s of the whole job, inputs resident in HBM, K steps timed
           with CUDA events on the executor's stream, max over ranks.
e2e        same metric through the public API (SlimPipeStep.step) with the
           tokens/targets copied from pinned host memory each step and the
           loss read back each step.
roofline   the dominant kernel (sliced attention backward, K2): algorithmic
           FLOPs per launch / mean launch time (CUDA events on the launching
           stream) vs the measured sustained bf16 peak.
cpu_baseline  the reference's own chunk_attention (oracle/_ref, fp64, all host
           threads) on a bounded sample of the same attention, extrapolated
           to the step's model FLOPs.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os

# one hardware work queue per CUDA stream (the executor runs up to ten per
# rank; shared queues let a waiting stream stall unrelated ones) — before the
# CUDA context exists
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return dict(PEAKS_FALLBACK), "fallback"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--model", choices=["c2", "c3", "c4"], default="c2",
                    help="BASELINE.json layer shapes: c2 Llama-7B, c3 Llama-13B, c4 Llama-70B (GQA 64/8)")
    ap.add_argument("--layers", type=int, default=None, help="default: c2 8, c3 8, c4 2")
    ap.add_argument("--seq-len", type=int, default=None, help="default: c2 128K, c3 256K, c4 1M")
    ap.add_argument("--slices", type=int, default=None, help="default: c2 8, c3 16, c4 32")
    ap.add_argument("--microbatches", type=int, default=None, help="default: c2 4, c3 4, c4 1")
    ap.add_argument("--recompute", choices=["auto", "selective", "full"], default="auto",
                    help="selective: the forward stashes attention O/LSE, the backward recomputes the rest; "
                         "auto: selective when the stash fits in HBM")
    ap.add_argument("--exchange", choices=["off", "on", "early"], default="off",
                    help="attention workload redistribution (reference ExchangeMode); no effect at PP=1")
    ap.add_argument("--vocab-parallel", action="store_true",
                    help="shard the LM head and cross entropy over all stages (PP>1; SURVEY §8f rank 1)")
    ap.add_argument("--offload", action="store_true",
                    help="activation offload: stage inputs + attention O/LSE in pinned host memory between F and BW")
    ap.add_argument("--exchange-min-chunks", type=int, default=0,
                    help="exchange placement: drop plan transfers that move fewer KV chunks")
    ap.add_argument("--exchange-skip-last", action="store_true",
                    help="exchange placement: drop plan transfers into the last stage (it also runs the LM head)")
    ap.add_argument("--dkv-bf16", action="store_true", help="dK/dV chunk accumulators stored in bf16 (half their HBM)")
    ap.add_argument("--interleave", type=int, default=1,
                    help="v stages per GPU (interleaved SlimPipe, even PP; SURVEY §8f rank 2)")
    ap.add_argument("--scenario", default=None,
                    help="reference scenario JSON (scenario.cpp schema) for the model/run shape; overrides --model etc.")
    ap.add_argument("--gantt", default=None,
                    help="write the measured last-step timeline in the reference's Gantt JSON format (rank 0)")
    ap.add_argument("--calibrate", default=None,
                    help="fit the reference CostModel to the measured last step and write the calibrated "
                         "simulate() prediction (exchange off/on/early) next to the measurement (rank 0)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


MODEL_NAMES = {"c2": ("c2 Llama-7B", "llama-7b-shapes"), "c3": ("c3 Llama-13B", "llama-13b-shapes"),
               "c4": ("c4 Llama-70B GQA", "llama-70b-shapes")}
DEPTH = {"c2": 8, "c3": 8, "c4": 2}  # reduced depth (BASELINE.json: "reduced depth")


def make_cfg(args, world):
    from paper_2504_14519_b200.runtime import StepConfig
    if args.scenario:  # a reference scenario file (scenario.cpp schema) names the whole step
        cfg = StepConfig.from_scenario(open(args.scenario).read())
        if cfg.pp != world:
            raise SystemExit(f"scenario pp={cfg.pp} but {world} rank(s) launched")
        return cfg
    base = getattr(StepConfig, args.model)()
    kw = {k: v for k, v in (("layers", args.layers or DEPTH[args.model]), ("seq_len", args.seq_len),
                            ("slices", args.slices), ("microbatches", args.microbatches)) if v is not None}
    return base.__class__(**{**base.__dict__, **kw, "pp": world, "exchange": args.exchange,
                             "recompute": args.recompute, "vocab_parallel": bool(args.vocab_parallel and world > 1),
                             "interleave": args.interleave if world > 1 else 1, "offload": bool(args.offload),
                             "dkv_bf16": bool(args.dkv_bf16), "exchange_min_chunks": args.exchange_min_chunks,
                             "exchange_skip_last": bool(args.exchange_skip_last)})


def workload_name(cfg, model="c2"):
    return (f"{MODEL_NAMES[model][0]} layer shapes x{cfg.layers} layers, {cfg.seq_len // 1024}K ctx, n={cfg.slices} slices, "
            f"m={cfg.microbatches}, PP={cfg.pp}, exchange={cfg.exchange}, recompute={cfg.recompute}"
            + (", vocab-parallel" if cfg.vocab_parallel else "") + (f", v={cfg.interleave}" if cfg.interleave > 1 else "")
            + (", activation offload" if cfg.offload else "") + (", bf16 dK/dV accumulators" if cfg.dkv_bf16 else "")
            + (f", exchange min {cfg.exchange_min_chunks} chunks" if cfg.exchange != "off" and cfg.exchange_min_chunks > 1 else "")
            + (", no exchange into the last stage" if cfg.exchange != "off" and cfg.exchange_skip_last else ""))


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx or None, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------- CPU baseline
def cpu_baseline(cfg, seconds: float):
    """Reference chunk_attention (fp64, all host threads) on a bounded sample
    of the step's attention, extrapolated to tokens/s of the full step."""
    threads = os.cpu_count() or 1
    ls, nch, d = 512, 4, 128
    flops_head = 4.0 * d * ls * ((nch - 1) * ls + (ls + 1) / 2.0)
    ref_so = ROOT / "oracle" / "_ref" / "libpipelab_ref.so"
    if ref_so.exists():
        lib = C.CDLL(str(ref_so))
        lib.ref_time_chunk_attention.restype = C.c_double
        lib.ref_time_chunk_attention.argtypes = [C.c_int] * 5 + [C.c_ulonglong]
        run = lambda heads: lib.ref_time_chunk_attention(heads, ls, nch, d, threads, 20240817)
        kind = "reference"
    else:  # C restatement (port)
        sys.path.insert(0, str(ROOT / "oracle"))
        import numpy as np
        import model_oracle as MO
        rng = np.random.default_rng(20240817)

        def run(heads):
            q = rng.uniform(-1, 1, (ls, heads, d)).astype(np.float32)
            k = rng.uniform(-1, 1, (nch * ls, heads, d)).astype(np.float32)
            t0 = time.perf_counter()
            MO.attn_fwd(q, k, k, ls)
            return time.perf_counter() - t0
        kind = "port"
    t = run(threads)  # calibrate
    heads = max(threads, int(threads * seconds / max(t, 1e-3)))
    t = run(heads)
    rate = heads * flops_head / t  # FLOP/s
    tok_s = cfg.microbatches * cfg.seq_len * rate / cfg.model_flops_per_step()
    sample = (f"{'reference' if kind == 'reference' else 'C-port'} chunk_attention fp64: {heads} heads x "
              f"(Ls={ls} causal over {nch} chunks, d={d}) = {heads * flops_head / 1e9:.1f} GFLOP in {t:.1f} s "
              f"({rate / 1e9:.2f} GFLOP/s on {threads} threads), extrapolated to the step's "
              f"{cfg.model_flops_per_step() / 1e15:.1f} PFLOP of model FLOPs")
    out = {"value": tok_s, "unit": "tokens/s", "cores": threads, "kind": kind, "sample": sample,
           "gflops": rate / 1e9, "seconds": t}
    try:
        out["details"] = cpu_details(cfg, threads, lib if kind == "reference" else None)
    except Exception as e:  # the headline baseline stands without the details
        out["details"] = {"error": str(e)}
    return out


def cpu_details(cfg, threads, ref_lib):
    """SURVEY §8(d)'s CPU-side numbers beside the headline sample: the
    reference's host planning of this step in ms (single thread), warm
    best-of-5 chunk_attention GFLOP/s at Ls 256/512/1024 (prefix <= 4 Ls,
    one head per thread), and the c1 tiny training step on the fp64 CPU
    oracle (tokens/s)."""
    d = {}
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O
    if ref_lib is not None:
        p = 8  # planned as the PP=8 configuration of this workload (BASELINE configs[1])
        t0 = time.perf_counter()
        O.ref_text("ref_schedule_json", 6, p, cfg.interleave, cfg.microbatches, cfg.slices)
        t1 = time.perf_counter()
        O.ref_text("ref_exchange_json", p, cfg.interleave, cfg.microbatches, cfg.slices, 2, 1.0)
        t2 = time.perf_counter()
        O.ref_text("ref_simulate_json", p, cfg.interleave, cfg.microbatches, cfg.slices, 0,
                   (C.c_double * 4)(1.0, 1e-3, 2.0, 1.0), (C.c_double * 2)(0.0, 0.0), cfg.seq_len, None)
        t3 = time.perf_counter()
        d["planning_ms"] = {"config": f"p={p} v={cfg.interleave} m={cfg.microbatches} n={cfg.slices}",
                            "gen_slimpipe + schedule_to_json": (t1 - t0) * 1e3,
                            "apply_exchange (early)": (t2 - t1) * 1e3, "simulate": (t3 - t2) * 1e3}
        att = {}
        for ls in (256, 512, 1024):
            best = None
            for _ in range(5):
                sec = ref_lib.ref_time_chunk_attention(threads, ls, 4, 128, threads, 20240817)
                best = sec if best is None else min(best, sec)
            fl = threads * 4.0 * 128 * ls * (3 * ls + (ls + 1) / 2.0)
            att[str(ls)] = fl / best / 1e9
        d["chunk_attention_gflops_best_of_5"] = att
    import numpy as np
    sys.path.insert(0, str(ROOT / "oracle"))
    import model_oracle as MO
    from paper_2504_14519_b200.runtime import StepConfig
    c1 = StepConfig.c1(microbatches=1, seq_len=1024, slices=4)
    rng = np.random.default_rng(0)
    W = {n: [rng.normal(0, 0.02, s) for _ in range(c1.layers)] for n, s in (
        ("attn_norm", (c1.hidden,)), ("wqkv", (3 * c1.hidden, c1.hidden)), ("wo", (c1.hidden, c1.hidden)),
        ("mlp_norm", (c1.hidden,)), ("wgu", (2 * c1.ffn_hidden, c1.hidden)), ("wd", (c1.hidden, c1.ffn_hidden)))}
    W["embedding"] = rng.normal(0, 0.02, (c1.vocab, c1.hidden))
    W["final_norm"] = np.ones(c1.hidden)
    W["head"] = rng.normal(0, 0.02, (c1.vocab, c1.hidden))
    tok = rng.integers(0, c1.vocab, (1, c1.seq_len))
    t0 = time.perf_counter()
    MO.Model(W, c1.heads, c1.kv_heads, c1.rope_theta, c1.norm_eps).step(tok, np.roll(tok, -1, axis=1), c1.slices)
    d["c1_oracle_step"] = {"tokens_per_s": c1.seq_len / (time.perf_counter() - t0),
                           "shape": "c1 layers (4 x h256, 4 heads), 1 microbatch of 1K tokens in 4 slices, fp64 numpy"}
    return d


def run_reference(args):
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    cfg = make_cfg(args, world)
    if rank != 0:
        return 0
    vals = []
    for _ in range(args.warmup):
        cpu_baseline(cfg, min(3.0, args.cpu_seconds))
    base = None
    for _ in range(args.steps):
        base = cpu_baseline(cfg, args.cpu_seconds)
        vals.append(base["value"])
    value = sum(vals) / len(vals)
    ms = cfg.microbatches * cfg.seq_len / value * 1e3
    line = {"metric": "tokens/s", "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": workload_name(cfg, args.model), "global_batch": cfg.microbatches, "seq_len": cfg.seq_len,
                       "parallelism": f"pp{cfg.pp}"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": base["cores"], "kind": base["kind"],
                             "sample": base["sample"]},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------- ours
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}; using {world}", file=sys.stderr)
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2504_14519_b200 import native
    from paper_2504_14519_b200 import plan as PL
    from paper_2504_14519_b200.runtime import SlimPipeStep

    cfg = make_cfg(args, world)
    step = SlimPipeStep(cfg, rank, world)
    lib = native.lib()
    stream = torch.cuda.ExternalStream(step.stream_handle)

    rng = np.random.default_rng(1234)
    tok_host = torch.from_numpy(rng.integers(0, cfg.vocab, (cfg.microbatches, cfg.seq_len), dtype=np.int32))
    tgt_host = torch.roll(tok_host, -1, dims=1)
    tok_pin = tok_host.pin_memory()
    tgt_pin = tgt_host.pin_memory()
    tok_dev = tok_host.cuda()
    tgt_dev = tgt_host.cuda()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    for _ in range(args.warmup):
        step.step_async(tok_dev.data_ptr(), tgt_dev.data_ptr())
    step.sync()
    torch.cuda.synchronize()

    # ---- timed region (value): device-resident inputs
    clocks = ClockSampler()
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    launches0 = lib.sp_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step.step_async(tok_dev.data_ptr(), tgt_dev.data_ptr())
    ev1.record(stream)
    step.sync()
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = lib.sp_launch_count() - launches0
    ms_total = max_over_ranks(ev0.elapsed_time(ev1))
    ms_step = ms_total / args.steps
    tokens_per_step = cfg.microbatches * cfg.seq_len
    value = tokens_per_step * args.steps / (ms_total / 1e3)

    # last timed step: per-pass busy (bubble) and attention kernel timings
    step_ms, passes = step.timeline()
    per_dev = [passes]
    clock_check = None
    if world > 1 and (args.gantt or args.calibrate):
        per_dev = [None] * world
        dist.all_gather_object(per_dev, passes)
        # each rank's spans are relative to its own step start (CUDA events are
        # per device, and the GPUs' global timers measured hundreds of ms apart),
        # so place rank r on rank 0's clock by its first dependency: its first
        # pass starts when the previous stage's first pass has delivered its
        # output (the rank was waiting for it; the 128 MB message is < 1 ms)
        offsets = [0.0]
        for r in range(1, world):
            prev_end = min(per_dev[r - 1], key=lambda x: x[1])[2] + offsets[r - 1]
            offsets.append(prev_end - min(per_dev[r], key=lambda x: x[1])[1])
        per_dev = [[(i, s + offsets[r], e + offsets[r]) for i, s, e in spans] for r, spans in enumerate(per_dev)]
        clock_check = {"method": "first-pass dependency", "offsets_ms": offsets}
    calib = None
    if args.calibrate and rank == 0 and not cfg.vocab_parallel:
        from paper_2504_14519_b200 import calibrate as CAL
        calib = CAL.predict(world, cfg.interleave, cfg.microbatches, cfg.slices, cfg.seq_len, per_dev)
        calib["workload"] = workload_name(cfg, args.model)
        with open(args.calibrate, "w") as f:
            json.dump(calib, f, indent=1)
    if args.gantt:  # measured timeline in the reference's Gantt schema (gantt.cpp:52-106)
        from paper_2504_14519_b200 import plan as P
        if rank == 0:
            with open(args.gantt, "w") as f:
                f.write(P.gantt_measured_text(world, cfg.interleave, cfg.microbatches, cfg.slices, per_dev,
                                              cfg.vocab_parallel, cfg.seq_len))
            with open(args.gantt + ".metrics.json", "w") as f:  # reference metric definitions, measured
                json.dump(P.metrics_measured(world, cfg.interleave, cfg.microbatches, cfg.slices, per_dev,
                                             cfg.vocab_parallel, cfg.seq_len), f, indent=1)
    busy = sum(e - s for _, s, e in passes)
    makespan = max_over_ranks(step_ms)
    busy_all = sum_over_ranks(busy)
    bubble = (world * makespan - busy_all) / busy_all if busy_all > 0 else 0.0
    at = step.attn_stats()
    cs = step.comm_stats()
    mem = step.memory()
    at_tot = {k: sum_over_ranks(float(v)) for k, v in at.items()}
    launches_all = int(sum_over_ranks(float(launches)))
    # cuBLASLt candidates timed at create (runtime warm-up): shapes where a
    # non-default algorithm won, and the per-call time saved
    plans = json.loads(native._json_call("sp_gemm_plans_json"))
    won = [q for q in plans if q["chosen"] != 0]
    gemm_tune = {"shapes": len(plans), "non_default": len(won),
                 "ms_saved_per_call": sum(q["ms_first"] - q["ms_chosen"] for q in won)}
    # stage P2P over NVLink: fastest message of any rank (link rate once the
    # receive is posted) and the mean over all stage sends of the last step
    link = None
    if world > 1:
        msg_b = cfg.slice_len * cfg.hidden * 2
        fastest = -max_over_ranks(-cs["fastest_ms"] if cs["messages"] else -1e30)
        n_msg, sum_ms = sum_over_ranks(cs["messages"]), sum_over_ranks(cs["send_ms"])
        link = {"message_bytes": msg_b, "messages_per_step": int(n_msg),
                "fastest_gbs": msg_b / (fastest / 1e3) / 1e9 if fastest > 0 else None,
                "mean_gbs": n_msg * msg_b / (sum_ms / 1e3) / 1e9 if sum_ms > 0 else None,
                "peak_gbs": 900.0, "timer": "CUDA events around each stage send on its stream (incl. waits)"}

    # ---- e2e through the public API: pinned host inputs, loss read back every step
    e2e = None
    if not args.no_e2e:
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        loss, losses = 0.0, []
        for _ in range(args.steps):
            loss = step.step(tok_pin.numpy(), tgt_pin.numpy())
            losses.append(loss)
        torch.cuda.synchronize()
        barrier()
        wall = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": tokens_per_step * args.steps / wall, "unit": "tokens/s",
               "h2d_bytes_per_step": 2 * tokens_per_step * 4, "d2h_bytes_per_step": 4 * world,
               "timer": "host wall clock around SlimPipeStep.step (includes H2D/D2H), max over ranks"}
        if world > 1:
            t = torch.tensor(losses, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.SUM)  # only the last stage is non-zero
            losses = [float(x) for x in t.tolist()]
            loss = losses[-1]
        e2e["loss"] = loss
        # sanity of the training signal: finite, and an optimizer step per call
        # (the first timed steps follow the warm-up's updates); ln V = the
        # loss of a uniform prediction
        e2e["losses"] = losses
        e2e["ln_vocab"] = float(np.log(cfg.vocab))
        e2e["loss_finite"] = bool(all(np.isfinite(losses)))

    peaks, peak_src = load_peaks()
    peak_tf = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    mfu = cfg.model_flops_per_step() / (ms_step / 1e3) / world / (peak_tf * 1e12)
    mfu_nominal = cfg.model_flops_per_step() / (ms_step / 1e3) / world / 2.25e15
    # dominant kernel: whichever attention direction has the larger total time
    kind = "bwd" if at_tot["bwd_ms"] >= at_tot["fwd_ms"] else "fwd"
    n_l = max(1.0, at_tot[f"{kind}_launches"])
    achieved = (at_tot[f"{kind}_flops"] / n_l) / (at_tot[f"{kind}_ms"] / n_l / 1e3) / 1e12
    traffic = None
    prof = ROOT / "profiles" / "roofline_traffic.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get(f"attn_{kind}", {}).get("dram_bytes_per_launch")
    # activation memory: arena slots x slot bytes (x stash + per-layer K/V), max over ranks
    arena_gb = max_over_ranks(mem["slots"] * mem["slot_bytes"] / 1e9)
    dkv_gb = cfg.layers // world * cfg.seq_len * 2 * cfg.kv_heads * cfg.head_dim * (2 if cfg.dkv_bf16 else 4) / 1e9
    mm = PL.activation_bytes(PL.ModelShape(cfg.layers, cfg.hidden, cfg.ffn_hidden, cfg.heads, cfg.kv_heads,
                                           cfg.vocab), 1, 1, world, 1, cfg.seq_len, cfg.microbatches, cfg.slices)
    ledger_gb = float(mm["slice_stage"]) * (cfg.slices + 2 * (world - 1)) / 1e9 if cfg.microbatches * cfg.slices >= \
        cfg.slices + 2 * (world - 1) else None
    offload_gb = max_over_ranks(mem["offload_host_bytes"] / 1e9)  # collectives: every rank, before the rank-0 line
    xst = step.exchange_stats() if cfg.exchange != "off" else None
    x_out = sum_over_ranks(xst["passes_out"]) if xst else 0
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_baseline(cfg, args.cpu_seconds)
            cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "details")}
        except Exception as e:  # never fail the bench line on the baseline leg
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": "tokens/s", "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic tokens, random-init weights",
            "config": {"workload": (f"scenario {os.path.basename(args.scenario)}: L={cfg.layers} h={cfg.hidden} "
                                    f"S={cfg.seq_len} n={cfg.slices} m={cfg.microbatches} PP={cfg.pp}"
                                    if args.scenario else workload_name(cfg, args.model)),
                       "model": "scenario" if args.scenario else MODEL_NAMES[args.model][1], "layers": cfg.layers,
                       "global_batch": cfg.microbatches, "seq_len": cfg.seq_len, "slices": cfg.slices,
                       "parallelism": f"pp{world}", "exchange": cfg.exchange, "vocab_parallel": cfg.vocab_parallel, "interleave": cfg.interleave,
                       "recompute": cfg.recompute if cfg.recompute != "auto" else f"auto->{mem['recompute']}",
                       "l2": "inputs larger than L2 (per-step working set tens of GB)"},
            "mfu": mfu, "mfu_nominal": mfu_nominal, "mfu_peak_tflops": peak_tf,
            "bubble_fraction": bubble,
            "timeline_clock": clock_check,
            "bubble_simulated_calibrated": ({k: v["bubble"] for k, v in calib["simulated"].items()}
                                            if calib else None),
            "peak_act_gb_per_gpu": arena_gb, "dkv_accum_gb_per_gpu": dkv_gb, "ledger_pred_gb_per_gpu": ledger_gb,
            "arena_slots": mem["slots"], "arena_high_water": mem["slots_high_water"],
            "offload_host_gb_per_gpu": offload_gb,
            "exchange_passes_sending": int(x_out),  # passes (all ranks) that ship attention work under the placement
            # logits workspace of the stage(s) holding the LM head: [Ls, V] fp32 logits + dlogits
            # (last stage), or the [Ls, V/p] shard (fp32 logits + bf16 dlogits) on every stage
            # under vocabulary parallelism (reference logits_bytes, workload.cpp:154-160)
            "logits_gb_per_gpu": (cfg.slice_len * (cfg.vocab // world) * 6 if cfg.vocab_parallel
                                  else cfg.slice_len * cfg.vocab * 8) / 1e9,
            "roofline": {"kernel": f"sp_attn_{kind} (sm_100a tcgen05)", "bound": "tensor", "achieved": achieved,
                         "peak": peak_tf, "unit": "TFLOP/s", "frac": achieved / peak_tf, "traffic": traffic,
                         "peak_source": f"{peak_src} bf16 sustained",
                         "attn_fwd_tflops": (at_tot["fwd_flops"] / max(1e-9, at_tot["fwd_ms"] / 1e3)) / 1e12,
                         "attn_bwd_tflops": (at_tot["bwd_flops"] / max(1e-9, at_tot["bwd_ms"] / 1e3)) / 1e12,
                         "attn_share_of_step": (at_tot["fwd_ms"] + at_tot["bwd_ms"]) / world / step_ms},
            "stage_p2p": link,
            "gemm_autotune": gemm_tune,
            "gpu_launches": launches_all,
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    step.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
