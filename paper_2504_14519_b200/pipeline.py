"""Per-rank communication programs of the B200 executor, derived from the
bit-exact plan (mirror of the order csrc/host/runtime.cpp posts NCCL calls).

Used by the multi-process CPU tests (gloo) to prove, before any GPU runs, that
every send has a matching receive in the same position on the peer — i.e.
that the P2P protocol the executor runs is deadlock-free for a given
(p, m, n, exchange mode):

* stage messages (schedule.cpp:102-130 cross-device edges): F(k,i,s) sends its
  output to s+1, F(k,i,s+1) receives it; BW(k,i,s+1) sends dX to s, BW(k,i,s)
  receives it.  One directional communicator each.
* exchange messages (simulator.cpp:56-108 tick plans): per pass and layer,
  the sender ships Q (+ dO/statistics in backward ticks) and its K/V chunks,
  the receiver returns the partial(s).  One communicator per tick class.
"""
from __future__ import annotations

import json

from . import plan as P


def device_passes(sched: dict, rank: int) -> list[dict]:
    return [sched["passes"][pid] | {"id": pid} for pid in sched["device_order"][rank]]


def stage_messages(sched: dict, rank: int) -> dict[str, list[tuple]]:
    """Ordered messages per (communicator, direction) for this rank."""
    p = sched["p"]
    stage = rank + 1
    out = {"fwd_send": [], "fwd_recv": [], "bwd_send": [], "bwd_recv": []}
    for ps in device_passes(sched, rank):
        key = (ps["microbatch"], ps["slice"])
        if ps["kind"] == "F":
            if stage > 1:
                out["fwd_recv"].append((rank - 1,) + key)
            if stage < p:
                out["fwd_send"].append((rank + 1,) + key)
        elif ps["kind"] == "BW":
            if stage < p:
                out["bwd_recv"].append((rank + 1,) + key)
            if stage > 1:
                out["bwd_send"].append((rank - 1,) + key)
    return out


def exchange_plan(sched: dict, ann: dict, rank: int) -> dict[int, dict]:
    """Per pass id of this rank: {'cls', 'out': [(peer, chunks)], 'in': [(peer, i_src, chunks)]}
    built exactly like Runtime::build_xplan."""
    me = rank + 1
    plan: dict[int, dict] = {}
    for tick in ann["ticks"]:
        devs = {dev: pid for dev, _load, pid in tick["in"]}
        for tr in tick["plan"]["transfers"]:
            sp, dp = devs.get(tr["src"]), devs.get(tr["dst"])
            if sp is None or dp is None:
                continue
            if tr["src"] == me:
                e = plan.setdefault(sp, {"cls": 1 - tick["fwd"], "out": [], "in": []})
                e["out"].append((tr["dst"] - 1, tuple(tr["chunks"])))
            if tr["dst"] == me:
                e = plan.setdefault(dp, {"cls": 1 - tick["fwd"], "out": [], "in": []})
                e["in"].append((tr["src"] - 1, sched["passes"][sp]["slice"], tuple(tr["chunks"])))
    return plan


def exchange_messages(sched: dict, ann: dict, rank: int, layers: int,
                      recompute: str = "selective") -> dict[int, list[tuple]]:
    """Ordered (op, peer, tag) per exchange communicator (class 0: forward
    ticks, 1: backward ticks) in the order this rank posts them.  Backward
    ticks carry the recompute's forward partials only under full recompute
    (selective recompute reuses the stashed attention output)."""
    xp = exchange_plan(sched, ann, rank)
    msgs: dict[int, list[tuple]] = {0: [], 1: []}
    for ps in device_passes(sched, rank):
        e = xp.get(ps["id"])
        if e is None:
            continue
        c = e["cls"]
        fwd = c == 0 or recompute == "full"
        phases = ([("fwd", l) for l in range(layers)] if fwd else []) + \
            ([("bwd", l) for l in reversed(range(layers))] if c else [])
        if e["in"]:  # receiver: posted at pass start, per layer and transfer: recv -> partial -> send back
            for phase, l in phases:
                for peer, _i_src, chunks in e["in"]:
                    msgs[c].append(("recv", peer, phase, l, len(chunks)))
                    msgs[c].append(("send", peer, phase, l, len(chunks)))
        if e["out"]:  # sender: per layer: ship to every receiver, then collect every partial
            for phase, l in phases:
                for peer, chunks in e["out"]:
                    msgs[c].append(("send", peer, phase, l, len(chunks)))
                for peer, chunks in e["out"]:
                    msgs[c].append(("recv", peer, phase, l, len(chunks)))
    return msgs


def schedule_and_annotation(p: int, m: int, n: int, mode: str) -> tuple[dict, dict]:
    sched = P.gen_slimpipe(p, 1, m, n)
    ann = json.loads(P.apply_exchange_text(p, 1, m, n, mode)) if mode != "off" else {"ticks": []}
    return sched, ann


def simulate_rendezvous(per_rank: list[list[tuple]]) -> None:
    """Run the ordered blocking send/recv programs of all ranks on one
    communicator (a send completes only together with the peer's matching
    receive at the head of its queue).  Raises AssertionError on deadlock."""
    heads = [0] * len(per_rank)
    progress = True
    while progress:
        progress = False
        for a, prog in enumerate(per_rank):
            if heads[a] >= len(prog):
                continue
            op = prog[heads[a]]
            if op[0] != "send":
                continue
            b = op[1]
            if heads[b] < len(per_rank[b]):
                peer_op = per_rank[b][heads[b]]
                if peer_op[0] == "recv" and peer_op[1] == a and peer_op[2:] == op[2:]:
                    heads[a] += 1
                    heads[b] += 1
                    progress = True
    stuck = [(r, per_rank[r][heads[r]]) for r in range(len(per_rank)) if heads[r] < len(per_rank[r])]
    assert not stuck, f"deadlock: {stuck[:4]}"


def check_pairwise(per_rank: list[list[tuple]]) -> None:
    """Every rank's ordered sends to peer q must equal q's ordered receives
    from it (tags included).  Raises AssertionError otherwise."""
    world = len(per_rank)
    for a in range(world):
        for b in range(world):
            if a == b:
                continue
            sends = [m[2:] for m in per_rank[a] if m[0] == "send" and m[1] == b]
            recvs = [m[2:] for m in per_rank[b] if m[0] == "recv" and m[1] == a]
            assert sends == recvs, f"rank {a}->{b}: {len(sends)} sends vs {len(recvs)} recvs"
