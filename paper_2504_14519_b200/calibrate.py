"""Calibrate the reference cost model from a measured step, and put the
reference simulator's prediction next to the measurement.

The reference prices passes with CostModel / pass_cost (workload.hpp:80-97,
workload.cpp:162-187):

    F(i)  = alpha * tok + beta * tok * (i * tok)          (kv = i slices)
    BW(i) = bwd_in * F(i) + bwd_w * alpha * tok

with tok = S / n.  A measured step gives the busy span of every pass
(SlimPipeStep.timeline(): CUDA events, after the pass's input arrived), so a
least-squares line through the forward spans against the slice index fixes
(alpha, beta) and one through the backward spans fixes (bwd_in, bwd_w).  The
calibrated costs then drive the reference simulate() (simulator.cpp:110-412)
on the same schedule, which predicts the makespan and bubble fraction
(:381-382) the executor should reach if the only losses were the schedule's
own — and, with exchange on / early, what the workload redistribution would
buy under the reference's model.

Everything here is host arithmetic on timelines; it runs without a GPU.
"""
from __future__ import annotations

import numpy as np

from . import plan as P


def _line(x, y):
    """Least squares y = a + b x; returns (a, b, max relative residual)."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    A = np.stack([np.ones_like(x), x], axis=1)
    (a, b), *_ = np.linalg.lstsq(A, y, rcond=None)
    res = float(np.max(np.abs(A @ np.array([a, b]) - y) / np.maximum(np.abs(y), 1e-30))) if len(y) else 0.0
    return float(a), float(b), res


def pass_table(p: int, v: int, m: int, n: int) -> dict[int, dict]:
    """pass id -> {kind, slice, stage, device} of gen_slimpipe (bit-exact host plan)."""
    return {q["id"]: q for q in P.gen_slimpipe(p, v, m, n)["passes"]}


def fit_costs(p: int, v: int, m: int, n: int, seq_len: int, per_device) -> dict:
    """(alpha, beta, bwd_in, bwd_w) of the reference CostModel from measured
    per-device spans [(pass_id, start_ms, end_ms), ...] (milliseconds)."""
    tab = pass_table(p, v, m, n)
    tok = seq_len // n
    fx, fy, bx, by = [], [], [], []
    for spans in per_device:
        for pid, s, e in spans:
            q = tab.get(int(pid))
            if q is None:
                continue
            (fx if q["kind"] == "F" else bx).append(q["slice"])
            (fy if q["kind"] == "F" else by).append(e - s)
    fa, fb, fres = _line(fx, fy)          # F(i) = fa + fb i
    ba, bb, bres = _line(bx, by)          # BW(i) = ba + bb i
    alpha = fa / tok
    beta = fb / (tok * tok)
    bwd_in = bb / fb if fb > 0 else 2.0
    bwd_w = ba / fa - bwd_in if fa > 0 else 1.0
    return {"alpha": alpha, "beta": beta, "bwd_in": bwd_in, "bwd_w": bwd_w, "tok": tok,
            "fwd_ms": [fa, fb], "bwd_ms": [ba, bb], "fit_residual": {"fwd": fres, "bwd": bres}}


def measured_bubble(per_device) -> tuple[float, float]:
    """(makespan, bubble) with the reference definition (p * makespan - sum busy)
    / sum busy (simulator.cpp:381-382) on measured spans, all on one clock
    whose zero is stage 1's step start (bench.py shifts each rank so that its
    first pass starts where the previous stage's first pass ended), as
    simulate() starts at 0."""
    busy = sum(e - s for spans in per_device for _, s, e in spans)
    mk = max(e for spans in per_device for _, _, e in spans)
    return mk, (len(per_device) * mk - busy) / busy if busy > 0 else 0.0


def predict(p: int, v: int, m: int, n: int, seq_len: int, per_device, modes=("off", "on", "early"),
            comm=(0.0, 0.0)) -> dict:
    """Calibrated simulate() beside the measured step."""
    fit = fit_costs(p, v, m, n, seq_len, per_device)
    cost = (fit["alpha"], fit["beta"], fit["bwd_in"], fit["bwd_w"])
    mk, bub = measured_bubble(per_device)
    out = {"p": p, "v": v, "m": m, "n": n, "seq_len": seq_len, "fit": fit,
           "measured": {"makespan_ms": mk, "bubble": bub}, "simulated": {}}
    for mode in modes:
        if p == 1 and mode != "off":
            continue
        sim = P.simulate(p, v, m, n, mode, cost=cost, comm=comm, seq_len=seq_len)
        out["simulated"][mode] = {"makespan_ms": sim["makespan"], "bubble": sim["bubble"]}
    return out
