"""The executor's exchange wiring (csrc/host/xplan.hpp, the exact per-pass
lists sp_runtime_create builds) checked against the reference's tick plans
(apply_exchange, simulator.cpp:56-108) on the CPU: every shipped transfer has
exactly one matching serve on the peer, the unfiltered wiring is the plan's
transfer set, and the placement filter (slimpipe.h exchange_min_chunks /
exchange_skip_last) only removes transfers — the same ones on every rank."""
from __future__ import annotations

from collections import Counter

import pytest

from paper_2504_14519_b200 import plan as P


def _wiring(p, m, n, mode, min_chunks=0, skip_last=False):
    """{(src rank, dst rank, src pass, chunks)} seen from the senders and from the receivers."""
    sched = P.gen_slimpipe(p, 1, m, n)
    sent, served = [], Counter()
    for r in range(p):
        for px in P.exchange_passes(p, m, n, mode, r, min_chunks, skip_last):
            assert sched["passes"][px["pass"]]["device"] == r + 1  # a pass of this rank
            base = 0
            for o in px["out"]:
                assert o["base"] == base  # partial-receive pool packed in plan order
                base += len(o["chunks"])
                sent.append((r, o["peer"], px["pass"], px["cls"], tuple(o["chunks"])))
            base = 0
            for i in px["in"]:
                assert i["base"] == base
                base += len(i["chunks"])
                served[(i["peer"], r, px["cls"], i["i_src"], tuple(i["chunks"]))] += 1
    return sched, sent, served


def _plan_transfers(p, m, n, mode):
    out = []
    for t in P.apply_exchange(p, 1, m, n, mode)["ticks"]:
        for tr in t["plan"]["transfers"]:
            out.append((tr["src"] - 1, tr["dst"] - 1, len(tr["chunks"]), tuple(tr["chunks"])))
    return out


@pytest.mark.parametrize("p,m,n", [(2, 2, 4), (2, 4, 8), (4, 2, 8), (4, 4, 8), (4, 4, 16)])
@pytest.mark.parametrize("mode", ["on", "early"])
@pytest.mark.parametrize("min_chunks,skip_last", [(0, False), (2, False), (0, True), (3, True)])
def test_every_shipped_transfer_has_one_serve(p, m, n, mode, min_chunks, skip_last):
    sched, sent, served = _wiring(p, m, n, mode, min_chunks, skip_last)
    # sender view (src, dst, pass, cls, chunks) vs receiver view (src, dst, cls, i_src, chunks)
    assert len(set(sent)) == len(sent)  # a (pass, peer) pair ships once
    assert Counter((s, d, c, sched["passes"][sp]["slice"], ch) for s, d, sp, c, ch in sent) == served
    for s, d, _, _, ch in sent:
        assert s != d and len(ch) >= max(1, min_chunks) and list(ch) == sorted(ch)
        assert not (skip_last and d == p - 1)


@pytest.mark.parametrize("p,m,n", [(2, 2, 4), (4, 4, 8), (4, 4, 16)])
@pytest.mark.parametrize("mode", ["on", "early"])
def test_unfiltered_wiring_is_the_plan_and_filters_only_remove(p, m, n, mode):
    plan = sorted((s, d, ch) for s, d, _, ch in _plan_transfers(p, m, n, mode))
    _, sent, _ = _wiring(p, m, n, mode)
    assert sorted((s, d, ch) for s, d, _, _, ch in sent) == plan
    for mc, sl in [(2, False), (0, True), (3, True)]:
        _, fs, _ = _wiring(p, m, n, mode, mc, sl)
        assert set(fs) == {x for x in sent if len(x[4]) >= mc and not (sl and x[1] == p - 1)}


def test_early_mode_ships_the_earliest_chunks_in_forward_ticks():
    """to_early_exchange (exchange.cpp:77-96), applied to forward ticks
    (simulator.cpp apply_exchange): consecutive chunks from 1 per sender pass."""
    _, sent, _ = _wiring(4, 4, 16, "early")
    fwd = [x for x in sent if x[3] == 0]
    assert fwd
    nxt = Counter()
    for s, d, sp, c, ch in sorted(fwd, key=lambda x: (x[2], x[1])):
        assert ch == tuple(range(nxt[sp] + 1, nxt[sp] + 1 + len(ch)))
        nxt[sp] += len(ch)


def test_rank_out_of_range_is_rejected():
    with pytest.raises(ValueError):
        P.exchange_passes(2, 2, 4, "on", 2)
