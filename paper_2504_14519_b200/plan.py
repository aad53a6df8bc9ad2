"""Python mirror of the pipelab planning API (reference
proj/include/pipelab/{schedule,exchange,simulator,workload}.hpp), backed by the
C++ implementation in libslimpipe.so.  Names and argument meanings follow the
reference; errors map std::invalid_argument -> ValueError and
std::runtime_error -> RuntimeError.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass
from fractions import Fraction

from . import native as N


def schedule_to_json(p: int, v: int, m: int, n: int, scheme: str = "slimpipe") -> str:
    """Byte-identical to reference schedule_to_json(generate(scheme, cfg))."""
    return N._json_call("sp_plan_schedule_json", N.SCHEMES[scheme], p, v, m, n)


def gen_slimpipe(p: int, v: int, m: int, n: int) -> dict:
    """reference schedule.cpp:248-279, returned as the parsed schedule JSON."""
    return json.loads(schedule_to_json(p, v, m, n, "slimpipe"))


def generate(scheme: str, p: int, v: int, m: int, n: int) -> dict:
    return json.loads(schedule_to_json(p, v, m, n, scheme))


def validate_schedule(p: int, v: int, m: int, n: int, mutation: int = 0) -> list[dict]:
    """Violations of gen_slimpipe(p,v,m,n) (optionally mutated, see slimpipe.h)."""
    return json.loads(N._json_call("sp_plan_validate_json", p, v, m, n, mutation))


def balance_tick(loads: list[int], devices: list[int] | None = None, early: bool = False) -> dict:
    devices = devices or list(range(1, len(loads) + 1))
    return json.loads(N._json_call("sp_plan_balance_json", N.arr(C.c_int64, loads), N.arr(C.c_int32, devices),
                                   len(loads), int(early)))


def to_early_exchange(loads: list[int], devices: list[int] | None = None) -> dict:
    return balance_tick(loads, devices, early=True)


def apply_exchange(p: int, v: int, m: int, n: int, mode: str = "on", beta_attn: float = 1.0) -> dict:
    return json.loads(N._json_call("sp_plan_exchange_json", p, v, m, n, N.MODES[mode], float(beta_attn)))


def apply_exchange_text(p: int, v: int, m: int, n: int, mode: str = "on", beta_attn: float = 1.0) -> str:
    return N._json_call("sp_plan_exchange_json", p, v, m, n, N.MODES[mode], float(beta_attn))


def exchange_passes(p: int, m: int, n: int, mode: str, rank: int, min_chunks: int = 0,
                    skip_last: bool = False) -> list[dict]:
    """The executor's per-pass exchange wiring of one rank (xplan.hpp): which
    passes ship work out and which serve a peer, after the placement filter."""
    return json.loads(N._json_call("sp_exchange_passes_json", p, m, n, N.MODES[mode], rank, int(min_chunks),
                                   int(skip_last)))


@dataclass
class ModelShape:
    layers: int
    hidden: int
    ffn_hidden: int
    heads: int
    query_groups: int
    vocab: int
    bytes_per_element: int = 2
    loss_bytes_per_element: int = 4

    def as_array(self):
        return [self.layers, self.hidden, self.ffn_hidden, self.heads, self.query_groups, self.vocab,
                self.bytes_per_element, self.loss_bytes_per_element]


CKPT = {"none": 0, "selective": 1, "full": 2}


def activation_bytes_text(model: ModelShape, tp: int, cp: int, pp: int, v: int, seq_len: int, m: int, n: int,
                          ckpt: str = "full", offload: float = 0.0) -> str:
    return N._json_call("sp_plan_activation_json", N.arr(C.c_int64, model.as_array()),
                        N.arr(C.c_int64, [tp, cp, pp, v]), N.arr(C.c_int64, [seq_len, m, n, CKPT[ckpt]]),
                        float(offload))


def activation_bytes(*args, **kw) -> dict[str, Fraction]:
    """reference workload.cpp:87-141; values as exact Fractions."""
    return {k: Fraction(v) for k, v in json.loads(activation_bytes_text(*args, **kw)).items()}


def exchange_volume(p: int, n: int, layers: int, mh: Fraction) -> dict[str, Fraction]:
    mh = Fraction(mh)
    d = json.loads(N._json_call("sp_plan_exchange_volume", p, n, layers, mh.numerator, mh.denominator))
    return {k: Fraction(v) for k, v in d.items()}


SCHEMES = {"gpipe": 0, "terapipe": 1, "1f1b": 2, "interleaved": 3, "zbv": 4, "vhalf": 5, "slimpipe": 6}


def analytics(scheme: str, p: int, m: int, n: int, v: int, ma: Fraction = Fraction(1)) -> dict:
    """Closed forms of analytics.hpp (reference analytics.cpp:11-112): memory
    multiplier, bubble bound, validity domain, SlimPipe attention asymptote and
    accumulated memory (for M_a = ma)."""
    ma = Fraction(ma)
    d = json.loads(N._json_call("sp_plan_analytics_json", SCHEMES[scheme], p, m, n, v, ma.numerator, ma.denominator))
    return {k: (Fraction(x) if isinstance(x, str) else x) for k, x in d.items()}


def simulate_text(p: int, v: int, m: int, n: int, mode: str = "off", cost=(1.0, 0.0, 2.0, 1.0), comm=(0.0, 0.0),
                  seq_len: int | None = None, mem_rats=None) -> str:
    seq_len = n if seq_len is None else seq_len
    mem = N.arr(C.c_int64, mem_rats) if mem_rats is not None else None
    return N._json_call("sp_plan_simulate_json", p, v, m, n, N.MODES[mode], N.arr(C.c_double, cost),
                        N.arr(C.c_double, comm), seq_len, mem)


def simulate(*args, **kw) -> dict:
    """reference simulator.cpp:110-412 on gen_slimpipe(p,v,m,n)."""
    return json.loads(simulate_text(*args, **kw))


def place_vocab_text(p: int, v: int, m: int, n: int, distribute: bool = True, alpha: float = 1.0,
                     beta: float = 1.0, seq_len: int | None = None) -> str:
    seq_len = n if seq_len is None else seq_len
    return N._json_call("sp_plan_vocab_json", p, v, m, n, int(distribute), float(alpha), float(beta), seq_len)


def place_vocab(*args, **kw) -> dict:
    """reference simulator.cpp:414-522 on gen_slimpipe(p,v,m,n): validity of the
    result and the per-device pass order ([kind, microbatch, slice, stage])."""
    return json.loads(place_vocab_text(*args, **kw))


# ---- scenario files and Gantt export ----------------------

def scenario_text(text: str) -> str:
    """reference scenario.cpp:72-193: strict parse + normalised re-serialisation
    (ValueError on unknown fields, bad values or malformed JSON)."""
    return N._json_call("sp_plan_scenario_json", text.encode())


def scenario(text: str) -> dict:
    return json.loads(scenario_text(text))


def gantt_text(p: int, v: int, m: int, n: int, mode: str = "off", cost=(1.0, 0.0, 2.0, 1.0), comm=(0.0, 0.0),
               seq_len: int | None = None, svg: bool = False) -> str:
    """reference gantt.cpp:52-106 on the simulated timeline of gen_slimpipe(p,v,m,n)."""
    seq_len = n if seq_len is None else seq_len
    return N._json_call("sp_plan_gantt_json", p, v, m, n, N.MODES[mode], N.arr(C.c_double, cost),
                        N.arr(C.c_double, comm), seq_len, int(svg))


def gantt_measured_text(p: int, v: int, m: int, n: int, per_device, vocab_parallel: bool = False,
                        seq_len: int = 1, svg: bool = False) -> str:
    """The same export for a measured step: per_device[d] = [(pass id, start ms,
    end ms), ...] as returned by SlimPipeStep.timeline() on rank d."""
    counts = [len(rows) for rows in per_device]
    flat = [e for rows in per_device for e in rows]
    return N._json_call("sp_plan_gantt_measured", p, v, m, n, int(vocab_parallel), seq_len,
                        N.arr(C.c_int32, counts), N.arr(C.c_int32, [int(e[0]) for e in flat]),
                        N.arr(C.c_double, [float(e[1]) for e in flat]), N.arr(C.c_double, [float(e[2]) for e in flat]),
                        int(svg))


def metrics_measured(p: int, v: int, m: int, n: int, per_device, vocab_parallel: bool = False,
                     seq_len: int = 1) -> dict:
    """The reference's metric definitions (simulator.cpp:348-409) on a measured
    step's per-device (pass id, start, end) spans."""
    counts = [len(rows) for rows in per_device]
    flat = [e for rows in per_device for e in rows]
    return json.loads(N._json_call("sp_plan_metrics_measured", p, v, m, n, int(vocab_parallel), seq_len,
                                   N.arr(C.c_int32, counts), N.arr(C.c_int32, [int(e[0]) for e in flat]),
                                   N.arr(C.c_double, [float(e[1]) for e in flat]),
                                   N.arr(C.c_double, [float(e[2]) for e in flat])))


def simulate_scenario(text: str) -> dict:
    """simulate() of a scenario file's run (gen_slimpipe(pp, stages_per_device,
    microbatches, slices) under its cost / comm model, sequence length and
    exchange mode; unit memory model): the predicted side of the same file
    StepConfig.from_scenario executes."""
    sc = scenario(text)
    if sc["scheme"] != "slimpipe":
        raise ValueError("simulate_scenario: scheme slimpipe only")
    pa, rn, co, cm = sc["parallelism"], sc["run"], sc["cost"], sc["comm"]
    return simulate(pa["pp"], pa["stages_per_device"], rn["microbatches"], rn["slices"], sc["exchange"],
                    (co["alpha_linear"], co["beta_attn"], co["bwd_input_mult"], co["bwd_weight_mult"]),
                    (cm["bandwidth"], cm["latency"]), rn["seq_len"])
