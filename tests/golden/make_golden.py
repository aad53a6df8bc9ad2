"""Regenerate tests/golden/* from the compiled reference (oracle/_ref).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
Every fixture is produced by the *unmodified* reference sources through
oracle/ref_shim.cpp; the product is never involved.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
import oracle_lib as O  # noqa: E402

SCHEMES = {"gpipe": 0, "terapipe": 1, "1f1b": 2, "interleaved_1f1b": 3, "zbv": 4, "vhalf": 5, "slimpipe": 6}


def schedule_grid():
    for sch, code in SCHEMES.items():
        for p in (1, 2, 4, 8):
            for v in (1, 2):
                for m in (1, 2, 4, 8):
                    for n in ((1, 2, 4, 8, 16, 32) if sch in ("slimpipe", "terapipe") else (1,)):
                        yield sch, code, p, v, m, n


def exchange_grid():
    for p in (2, 4, 8):
        for v in (1, 2):
            for m in (1, 2, 4):
                for n in (p, 2 * p, 4 * p):
                    for mode in (1, 2):
                        yield p, v, m, n, mode


def main():
    sched = {}
    full = {}
    for sch, code, p, v, m, n in schedule_grid():
        text = O.ref_text("ref_schedule_json", code, p, v, m, n)
        key = f"{sch}/p{p}v{v}m{m}n{n}"
        sched[key] = "error" if text.startswith('{"error') else hashlib.sha256(text.encode()).hexdigest()
        if sch == "slimpipe" and (p, v, m, n) in {(4, 1, 4, 8), (4, 2, 2, 8), (2, 1, 2, 4), (1, 1, 1, 1)}:
            full[key] = text
    (HERE / "schedule_sha256.json").write_text(json.dumps(sched, indent=0, sort_keys=True) + "\n")
    (HERE / "schedule_full.json").write_text(json.dumps(full) + "\n")

    ex = {}
    for p, v, m, n, mode in exchange_grid():
        text = O.ref_text("ref_exchange_json", p, v, m, n, mode, 1.0)
        ex[f"p{p}v{v}m{m}n{n}mode{mode}"] = hashlib.sha256(text.encode()).hexdigest()
    ex_full = {f"p{p}v{v}m{m}n{n}mode{mode}": O.ref_text("ref_exchange_json", p, v, m, n, mode, 1.0)
               for (p, v, m, n, mode) in [(2, 1, 2, 4, 1), (2, 1, 2, 4, 2), (4, 1, 4, 8, 1), (4, 1, 4, 8, 2),
                                          (8, 1, 4, 16, 1), (8, 1, 4, 16, 2), (8, 1, 4, 8, 2)]}
    (HERE / "exchange_sha256.json").write_text(json.dumps(ex, indent=0, sort_keys=True) + "\n")
    (HERE / "exchange_full.json").write_text(json.dumps(ex_full) + "\n")

    sims = {}
    cost = (C.c_double * 4)(1.0, 0.3, 2.0, 1.0)
    comm = (C.c_double * 2)(0.5, 0.1)
    for p, v, m, n in [(2, 1, 2, 4), (4, 1, 4, 8), (8, 1, 4, 8), (8, 1, 4, 16), (4, 2, 2, 8)]:
        for mode in (0, 1, 2):
            sims[f"p{p}v{v}m{m}n{n}mode{mode}"] = O.ref_text("ref_simulate_json", p, v, m, n, mode, cost, comm,
                                                             4 * n, None)
    (HERE / "simulate.json").write_text(json.dumps(sims) + "\n")

    # chunk_attention fixtures: inputs drawn uniform(-1,1) (verify.cpp:71-76),
    # bf16-representable so the same inputs can feed the GPU kernel.
    rng = np.random.default_rng(20240817)
    arrays = {}
    cases = [(128, 64, [128], True), (128, 64, [128, 128], True), (256, 128, [256, 256, 256], True),
             (128, 128, [128, 128], False), (64, 32, [16, 24, 40], True), (12, 8, [12], True)]
    for ci, (rows, d, sizes, causal) in enumerate(cases):
        total = sum(sizes)
        q, k, v = (rng.uniform(-1, 1, size=s).astype(np.float32) for s in ((rows, d), (total, d), (total, d)))
        # round to bf16 values
        q, k, v = (((x.view(np.uint32) + 0x8000) & 0xFFFF0000).view(np.float32) for x in (q, k, v))
        out, partial, mx, sm = O.ref_chunk_attention(q, k, v, sizes, causal)
        arrays.update({f"c{ci}_q": q, f"c{ci}_k": k, f"c{ci}_v": v, f"c{ci}_out": out, f"c{ci}_max": mx,
                       f"c{ci}_sum": sm, f"c{ci}_sizes": np.array(sizes), f"c{ci}_causal": np.array(causal)})
    np.savez_compressed(HERE / "chunk_attention.npz", **arrays)
    print("wrote", sorted(p.name for p in HERE.iterdir()))


# ---- SURVEY §8f fixtures: place_vocab, scenario files, Gantt export ----------

EXTRA_SCENARIOS = [
    "{}",
    '{"model":{"layers":8,"hidden":4096,"ffn":11008,"heads":32,"query_groups":32,"vocab":32000},'
    '"parallelism":{"pp":2},"run":{"seq_len":131072,"microbatches":4,"slices":8,"checkpointing":"selective"},'
    '"scheme":"slimpipe","exchange":"off","seed":7}',
    '{"model":{"layers":80,"hidden":8192,"ffn":28672,"heads":64,"query_groups":8,"vocab":128000},'
    '"parallelism":{"tp":8,"pp":8,"stages_per_device":2},"run":{"seq_len":1048576,"microbatches":2,"slices":32,'
    '"checkpointing":"full","offload_ratio":0.25,"vocab_parallel":true},"cost":{"alpha_linear":1.5,'
    '"beta_attn":2.5e-07,"vocab_gemm":0.125},"comm":{"bandwidth":4.5e11,"latency":1e-05},'
    '"coeffs":{"key":0.5,"value":0.5},"exchange":"on+early","seed":123}',
    '{"model":{"layerz":1}}',
    '{"parallelism":{"pp":4},"run":{"slices":6}}',
]


def extras():
    out = {"scenario": {}, "gantt": {}, "gantt_full": {}, "vocab": {}}
    for t in EXTRA_SCENARIOS:
        r = O.ref_text("ref_scenario_json", t.encode())
        out["scenario"][t] = "error" if r.startswith('{"error') else r
    cost = (C.c_double * 4)(1.0, 1e-3, 2.0, 1.0)
    comm = (C.c_double * 2)(1e3, 0.5)
    for p, v, m, n in [(1, 1, 2, 4), (2, 1, 2, 4), (2, 2, 2, 4), (4, 1, 4, 8), (4, 2, 2, 8), (8, 1, 4, 16)]:
        for mode in ((0, 1) if v == 1 else (0,)):
            for svg in (0, 1):
                text = O.ref_text("ref_gantt_json", p, v, m, n, mode, cost, comm, 1024 * n, svg)
                key = f"p{p}v{v}m{m}n{n}mode{mode}svg{svg}"
                out["gantt"][key] = hashlib.sha256(text.encode()).hexdigest()
                if (p, v, m, n, mode) == (2, 1, 2, 4, 0):
                    out["gantt_full"][key] = text
    for p, m, n in [(2, 2, 4), (2, 4, 8), (4, 2, 8), (8, 2, 16)]:
        S = 1024 * n
        for raw in (0, 1):
            a, b = (1.0, 1.0) if raw else (1.0 / S, 1.0 / S ** 2)
            text = O.ref_text("ref_vocab_json", p, 1, m, n, 1, a, b, 4096 if raw else S)
            out["vocab"][f"p{p}m{m}n{n}raw{raw}"] = hashlib.sha256(text.encode()).hexdigest()
    (HERE / "planning_extras.json").write_text(json.dumps(out, indent=0, sort_keys=True) + "\n")


if __name__ == "__main__":
    if sys.argv[1:] == ["--extras"]:
        extras()
    else:
        main()
        extras()
