"""Pin of the timed stream model (scripts/exchange_timed_model.py) against
a measured 4-GPU step: fed the per-pass spans of the measured exchange-off
step (profiles/r02_xp/c2_off.gantt.json), its own off prediction must give
back the measured makespan, and with the exchange's transfers dispatched
behind the running attention kernel (equal stream priorities, as built) it
must not predict a gain — the sign measured on hardware."""
from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "scripts"))

import exchange_timed_model as TM  # noqa: E402

GANTT = ROOT / "profiles" / "r02_xp" / "c2_off.gantt.json"
SIZES = (131072 // 8, 4096, 4096)


def _run(**kw):
    mk, dur, per_chunk = TM.measured(GANTT)
    ms, stuck = TM.simulate(4, 4, 8, dur=dur, per_chunk=per_chunk, layers=2, sizes=SIZES, gbs=500.0, **kw)
    assert not stuck
    return mk, ms


def test_off_prediction_reproduces_the_measured_step():
    mk, ms = _run(mode="off")
    assert abs(ms - mk) / mk < 0.02


def test_exchange_with_queued_dispatch_predicts_no_gain():
    _, off = _run(mode="off")
    _, filt = _run(mode="early", min_chunks=2, skip_last=True, gated=True)
    _, plan = _run(mode="early", gated=True)
    assert filt >= off * 0.995 and plan >= off  # measured: −7 % / −13 % tokens/s
