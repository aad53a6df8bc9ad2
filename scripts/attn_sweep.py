"""BASELINE config c5: sliced causal attention kernel sweep (head_dim 128,
32 heads, bf16): slice length Ls x prefix length P (P a multiple of Ls), K1
forward and K2 backward TFLOP/s against the measured bf16 peak.

The prefix K/V is one contiguous chunk of P + Ls keys (the kernels walk any
chunk table; a single chunk keeps the sweep within SP_MAX_CHUNKS at P = 1M).
FLOPs: forward 4·d·Ls·(P + (Ls+1)/2)·a, backward 2.5x.
Writes gpurun_out/attn_sweep.json."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2504_14519_b200 import ops  # noqa: E402

HEADS, D = 32, 128
PEAK = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json"))).get(
    "bf16_tflops_sustained", 1412.3) if os.path.exists(
    os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")) else 1412.3


def timed(fn, iters):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


rows = []
for Ls in (4096, 8192, 16384, 32768, 65536):
    for P in (0, 65536, 131072, 262144, 524288, 1048576):
        if P % Ls:
            continue
        T = P + Ls
        q = torch.randn(Ls, HEADS * D, device="cuda", dtype=torch.bfloat16)
        kp = torch.randn(T, HEADS * D, device="cuda", dtype=torch.bfloat16)
        vp = torch.randn(T, HEADS * D, device="cuda", dtype=torch.bfloat16)
        do = torch.randn(Ls, HEADS * D, device="cuda", dtype=torch.bfloat16)
        fl = 4.0 * D * Ls * (P + (Ls + 1) / 2) * HEADS
        iters = max(1, min(10, int(2e15 / fl)))
        o, lse = ops.attn_fwd(q, kp, vp, [0], T, HEADS, HEADS, True)
        ms_f = timed(lambda: ops.attn_fwd(q, kp, vp, [0], T, HEADS, HEADS, True), iters)
        dq = torch.zeros(Ls, HEADS * D, device="cuda")
        dk = torch.zeros(T, HEADS * D, device="cuda")
        dv = torch.zeros_like(dk)
        ws = torch.empty(2 * HEADS * Ls, device="cuda")
        ms_b = timed(lambda: ops.attn_bwd(q, kp, vp, [0], T, HEADS, HEADS, True, o, lse, do, dq, dk, dv, [0], ws), iters)
        r = {"Ls": Ls, "P": P, "fwd_ms": ms_f, "bwd_ms": ms_b, "fwd_tflops": fl / ms_f / 1e9,
             "bwd_tflops": 2.5 * fl / ms_b / 1e9}
        r["fwd_frac"] = r["fwd_tflops"] / PEAK
        r["bwd_frac"] = r["bwd_tflops"] / PEAK
        rows.append(r)
        print(f"Ls={Ls:6d} P={P:8d}  fwd {r['fwd_tflops']:6.0f} TF/s ({r['fwd_frac']:.2f})  "
              f"bwd {r['bwd_tflops']:6.0f} TF/s ({r['bwd_frac']:.2f})", flush=True)
        del q, kp, vp, do, dq, dk, dv, ws, o, lse
        torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump({"peak_tflops": PEAK, "heads": HEADS, "head_dim": D, "rows": rows}, open("gpurun_out/attn_sweep.json", "w"),
          indent=1)
