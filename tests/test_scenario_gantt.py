"""Scenario files and Gantt export: the reference's
scenario schema (scenario.cpp:72-193) drives both the planner and the GPU
step; the reference's Gantt format (gantt.cpp:52-106) carries simulated and
measured timelines.  Parity is byte-for-byte against the compiled reference
(oracle/_ref) where it is available."""
import ctypes as C
import json

import pytest

from paper_2504_14519_b200 import plan as P
from paper_2504_14519_b200.runtime import StepConfig
import oracle_lib as O

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="compiled reference not available")

SCENARIOS = [
    "{}",
    '{"model":{"layers":8,"hidden":4096,"ffn":11008,"heads":32,"query_groups":32,"vocab":32000},'
    '"parallelism":{"pp":2},"run":{"seq_len":131072,"microbatches":4,"slices":8,"checkpointing":"selective"},'
    '"scheme":"slimpipe","exchange":"off","seed":7}',
    '{"model":{"layers":80,"hidden":8192,"ffn":28672,"heads":64,"query_groups":8,"vocab":128000,'
    '"bytes_per_element":2,"loss_bytes_per_element":4},"parallelism":{"tp":8,"cp":1,"dp":1,"ep":1,"pp":8,'
    '"stages_per_device":2},"run":{"seq_len":1048576,"microbatches":2,"slices":32,"checkpointing":"full",'
    '"offload_ratio":0.25,"vocab_parallel":true},"scheme":"slimpipe","cost":{"alpha_linear":1.5,'
    '"beta_attn":2.5e-07,"bwd_input_mult":2,"bwd_weight_mult":1,"vocab_gemm":0.125},"comm":{"bandwidth":4.5e11,'
    '"latency":1e-05},"coeffs":{"attn_input":1,"query":1,"key":0.5,"value":0.5,"attn_output":1,"norm_outputs":2,'
    '"mlp_input":1,"mlp_gate_up":2,"mlp_act":1},"exchange":"on+early","seed":123}',
    '{"parallelism":{"pp":4},"run":{"seq_len":8192,"slices":8},"scheme":"1f1b","exchange":"on"}',
]
BAD = ['{"model":{"layerz":1}}', '{"x":1}', '{"run":{"checkpointing":"some"}}', '{"scheme":"foo"}',
       '{"model":3}', '{"parallelism":{"pp":4},"run":{"slices":6}}', '{"exchange":"sideways"}']


@needs_ref
@pytest.mark.parametrize("text", SCENARIOS)
def test_scenario_roundtrip_matches_reference(text):
    mine = P.scenario_text(text)
    assert mine == O.ref_text("ref_scenario_json", text.encode())
    assert P.scenario_text(mine) == mine  # normalised form is a fixed point


@pytest.mark.parametrize("text", BAD + ["{not json", '{"run":{"vocab_parallel":3}}'])
def test_scenario_rejects_like_reference(text):
    with pytest.raises(ValueError):
        P.scenario_text(text)
    if O.ref_available():
        assert O.ref_text("ref_scenario_json", text.encode()).startswith('{"error"')


def test_scenario_drives_the_step_config():
    cfg = StepConfig.from_scenario(SCENARIOS[1])
    assert (cfg.layers, cfg.hidden, cfg.ffn_hidden, cfg.heads, cfg.kv_heads, cfg.vocab) == (8, 4096, 11008, 32, 32,
                                                                                            32000)
    assert (cfg.seq_len, cfg.microbatches, cfg.slices, cfg.pp, cfg.interleave) == (131072, 4, 8, 2, 1)
    assert cfg.recompute == "selective" and cfg.exchange == "off" and cfg.seed == 7
    assert cfg == StepConfig.c2(pp=2, recompute="selective", seed=7)
    for bad in (SCENARIOS[2], SCENARIOS[3]):  # tp=8 / offload, scheme 1f1b: not on the executed path
        with pytest.raises(ValueError):
            StepConfig.from_scenario(bad)


GRID = [(p, v, m, n, mode, beta) for p in (1, 2, 4) for v in (1, 2) for m in (1, 2, 4) for n in (4, 8)
        for mode in ("off", "on") for beta in (0.0, 1e-3) if n % p == 0 and not (v > 1 and mode != "off")]


@needs_ref
def test_gantt_json_and_svg_match_reference():
    n = 0
    for p, v, m, ns, mode, beta in GRID:
        cost, comm = (1.0, beta, 2.0, 1.0), (1e3, 0.5)
        for svg in (0, 1):
            mine = P.gantt_text(p, v, m, ns, mode, cost, comm, 1024 * ns, bool(svg))
            ref = O.ref_text("ref_gantt_json", p, v, m, ns, P.N.MODES[mode], (C.c_double * 4)(*cost),
                             (C.c_double * 2)(*comm), 1024 * ns, svg)
            assert mine == ref, (p, v, m, ns, mode, beta, svg)
            n += 1
    assert n > 100


def _synthetic_measured(p, v, m, n):
    """Per-device (pass id, start, end) spans: the simulated timeline, jittered
    as a CUDA-event timeline would be (ms, arbitrary offsets)."""
    sim = P.simulate(p, v, m, n, "off", (1.0, 1e-3, 2.0, 1.0), (0.0, 0.0), 1024 * n)
    rows = []
    for d, dev in enumerate(sim["timeline"]):
        rows.append([(pid, 0.37 * d + 1.001 * s, 0.37 * d + 1.003 * e) for pid, s, e in dev])
    return rows


@needs_ref
@pytest.mark.parametrize("p,v,m,n", [(1, 1, 2, 4), (2, 1, 2, 4), (4, 1, 3, 8), (2, 2, 2, 4), (4, 2, 2, 8)])
def test_gantt_of_measured_timeline_matches_reference(p, v, m, n):
    rows = _synthetic_measured(p, v, m, n)
    counts = [len(r) for r in rows]
    flat = [e for r in rows for e in r]
    for svg in (0, 1):
        mine = P.gantt_measured_text(p, v, m, n, rows, svg=bool(svg))
        ref = O.ref_text("ref_gantt_measured", p, v, m, n, (C.c_int32 * len(counts))(*counts),
                         (C.c_int32 * len(flat))(*[e[0] for e in flat]), (C.c_double * len(flat))(*[e[1] for e in flat]),
                         (C.c_double * len(flat))(*[e[2] for e in flat]), svg)
        assert mine == ref


def test_gantt_of_measured_timeline_rows_and_bounds():
    rows = _synthetic_measured(2, 1, 2, 4)
    g = json.loads(P.gantt_measured_text(2, 1, 2, 4, rows))
    assert g["devices"] == 2 and len(g["rows"]) == 2 and g["transfers"] == []
    assert g["makespan"] == max(e[2] for r in rows for e in r)
    assert [len(r) for r in g["rows"]] == [len(r) for r in rows] == [16, 16]
    assert {x["kind"] for r in g["rows"] for x in r} == {"F", "BW"}
    with pytest.raises(ValueError):
        P.gantt_measured_text(2, 1, 2, 4, [[(999, 0.0, 1.0)], []])


def test_bundled_scenarios_are_the_bench_configs():
    """scenarios/*.json (normalised form) describe bench.py's c2 step at PP=1/2/4."""
    from pathlib import Path
    root = Path(__file__).resolve().parents[1] / "scenarios"
    for pp in (1, 2, 4):
        text = (root / f"c2_llama7b_shapes_128k_pp{pp}.json").read_text()
        assert P.scenario_text(text) + "\n" == text
        assert StepConfig.from_scenario(text) == StepConfig.c2(pp=pp, recompute="selective")


# ---- the same parity against committed fixtures (no reference needed) --------

def _extras():
    import hashlib
    from pathlib import Path
    g = json.loads((Path(__file__).resolve().parent / "golden" / "planning_extras.json").read_text())
    return g, (lambda s: hashlib.sha256(s.encode()).hexdigest())


def test_scenarios_match_golden():
    g, _ = _extras()
    assert len(g["scenario"]) == 5
    for text, ref in g["scenario"].items():
        if ref == "error":
            with pytest.raises(ValueError):
                P.scenario_text(text)
        else:
            assert P.scenario_text(text) == ref


def test_gantt_matches_golden():
    g, sha = _extras()
    cost, comm = (1.0, 1e-3, 2.0, 1.0), (1e3, 0.5)
    for key, digest in g["gantt"].items():
        p, rest = key[1:].split("v", 1)
        v, rest = rest.split("m", 1)
        m, rest = rest.split("n", 1)
        n, rest = rest.split("mode", 1)
        mode, svg = rest.split("svg")
        p, v, m, n, mode, svg = map(int, (p, v, m, n, mode, svg))
        text = P.gantt_text(p, v, m, n, ["off", "on", "early"][mode], cost, comm, 1024 * n, bool(svg))
        assert sha(text) == digest, key
        if key in g["gantt_full"]:
            assert text == g["gantt_full"][key]
    assert len(g["gantt"]) == 20


def test_place_vocab_matches_golden():
    g, sha = _extras()
    for key, digest in g["vocab"].items():
        p, rest = key[1:].split("m", 1)
        m, rest = rest.split("n", 1)
        n, raw = rest.split("raw")
        p, m, n, raw = map(int, (p, m, n, raw))
        S = 1024 * n
        a, b = (1.0, 1.0) if raw else (1.0 / S, 1.0 / S ** 2)
        assert sha(P.place_vocab_text(p, 1, m, n, True, a, b, 4096 if raw else S)) == digest, key


@pytest.mark.parametrize("p,v,m,n", [(2, 1, 2, 4), (4, 1, 4, 8), (4, 2, 2, 8), (8, 1, 4, 16)])
def test_metrics_of_a_measured_timeline_use_the_reference_definitions(p, v, m, n):
    """Fed simulate()'s own timeline as if it were measured, the measured-run
    metrics reproduce simulate()'s makespan, bubble, busy time and phases
    (simulator.cpp:348-409) — the definitions bench.py's timelines go through."""
    sim = P.simulate(p, v, m, n, "off", (1.0, 1e-3, 2.0, 1.0), (0.0, 0.0), 1024 * n)
    rows = [[tuple(e) for e in dev] for dev in sim["timeline"]]
    got = P.metrics_measured(p, v, m, n, rows)
    assert got["makespan"] == pytest.approx(sim["makespan"], rel=1e-12)
    assert got["bubble"] == pytest.approx(sim["bubble"], rel=1e-9, abs=1e-12)
    assert got["busy"] == pytest.approx(sim["busy"], rel=1e-12)
    for a, b in zip(got["phases"], sim["phases"]):
        assert a == pytest.approx(b, rel=1e-9, abs=1e-9)


def test_one_scenario_file_drives_simulate_and_the_step():
    from pathlib import Path
    text = (Path(__file__).resolve().parents[1] / "scenarios" / "c2_llama7b_shapes_128k_pp2.json").read_text()
    cfg = StepConfig.from_scenario(text)
    sim = P.simulate_scenario(text)
    direct = P.simulate(cfg.pp, cfg.interleave, cfg.microbatches, cfg.slices, cfg.exchange, (1.0, 0.0, 2.0, 1.0),
                        (0.0, 0.0), cfg.seq_len)
    assert sim == direct and len(sim["busy"]) == cfg.pp


def test_scenario_offload_ratio_runs_the_executor_offload():
    """offload_ratio > 0 (reference workload.cpp:130-132) selects the
    executor's activation offload (everything but K/V to the host)."""
    text = SCENARIOS[1].replace('"checkpointing":"selective"}', '"checkpointing":"selective","offload_ratio":0.5}')
    cfg = StepConfig.from_scenario(text)
    assert cfg.offload and cfg.to_c(0).offload == 1
    assert not StepConfig.from_scenario(SCENARIOS[1]).offload
