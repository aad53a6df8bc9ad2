"""Where could the exchange's moved attention land for free?  Reads a measured
exchange-off Gantt (bench.py --gantt; ranks on one clock) and the reference
plan's transfers (apply_exchange, simulator.cpp:56-108), and for every
transfer reports the receiving GPU's idle time inside the sending pass's
window — the time the moved partial could run without delaying the receiver.
Moved work is estimated as the sender pass's duration x (chunks moved /
chunks the pass attends) x the attention share of the pass (--attn-share,
from the bench line's roofline.attn_share_of_step).  Also reports the same
for the best receiver per sender pass (any GPU idle in that window), the
upper bound for a placement that pairs by measured idle time instead of
the tick column.

    python scripts/exchange_what_if.py GANTT.json P M N [--mode early] [--attn-share 0.73]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_14519_b200 import plan as P  # noqa: E402


def idle_in(row, a, b):
    """Idle time of one device's (sorted) passes inside [a, b]."""
    busy = 0.0
    for x in row:
        lo, hi = max(a, x["start"]), min(b, x["end"])
        if hi > lo:
            busy += hi - lo
    return (b - a) - busy


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("gantt")
    ap.add_argument("p", type=int)
    ap.add_argument("m", type=int)
    ap.add_argument("n", type=int)
    ap.add_argument("--mode", default="early")
    ap.add_argument("--attn-share", type=float, default=0.73)
    a = ap.parse_args()
    g = json.loads(Path(a.gantt).read_text())
    rows = [sorted(r, key=lambda x: x["start"]) for r in g["rows"]]
    span = {(x["kind"], x["microbatch"], x["slice"], x["stage"]): (x["start"], x["end"]) for r in rows for x in r}
    passes = P.gen_slimpipe(a.p, 1, a.m, a.n)["passes"]
    tot = dict(moved=0.0, fits_paired=0.0, fits_best=0.0, n=0)
    by_size = {}
    for t in P.apply_exchange(a.p, 1, a.m, a.n, a.mode)["ticks"]:
        pid = {d: q for d, _, q in t["in"]}
        for tr in t["plan"]["transfers"]:
            sp = passes[pid[tr["src"]]]
            s0, s1 = span[(sp["kind"], sp["microbatch"], sp["slice"], sp["stage"])]
            work = (s1 - s0) * a.attn_share * len(tr["chunks"]) / sp["slice"]
            free_paired = min(work, idle_in(rows[tr["dst"] - 1], s0, s1))
            free_best = max(min(work, idle_in(rows[d], s0, s1)) for d in range(a.p) if d != tr["src"] - 1)
            tot["moved"] += work
            tot["fits_paired"] += free_paired
            tot["fits_best"] += free_best
            tot["n"] += 1
            k = ("into last" if tr["dst"] == a.p else f"{len(tr['chunks'])} chunk(s)")
            b = by_size.setdefault(k, [0, 0.0, 0.0])
            b[0] += 1
            b[1] += work
            b[2] += free_paired
    # several senders can target one receiver's idle window at once: the
    # per-transfer amounts, capped per receiver by its idle time inside the
    # union of its senders' windows (no idle millisecond counted twice)
    union_cap = 0.0
    for d in range(a.p):
        wins, work_d = [], 0.0
        for t in P.apply_exchange(a.p, 1, a.m, a.n, a.mode)["ticks"]:
            pid = {dv: q for dv, _, q in t["in"]}
            for tr in t["plan"]["transfers"]:
                if tr["dst"] - 1 != d:
                    continue
                sp = passes[pid[tr["src"]]]
                s0, s1 = span[(sp["kind"], sp["microbatch"], sp["slice"], sp["stage"])]
                wins.append((s0, s1))
                w = (s1 - s0) * a.attn_share * len(tr["chunks"]) / sp["slice"]
                work_d += min(w, idle_in(rows[d], s0, s1))  # each transfer: its own window
        wins.sort()
        merged = []
        for w0, w1 in wins:
            if merged and w0 <= merged[-1][1]:
                merged[-1][1] = max(merged[-1][1], w1)
            else:
                merged.append([w0, w1])
        union_cap += min(work_d, sum(idle_in(rows[d], w0, w1) for w0, w1 in merged))
    out = {"gantt": a.gantt, "transfers": tot["n"], "moved_ms": round(tot["moved"]),
           "in_receiver_idle_capped_ms": round(union_cap),
           "in_receiver_idle_ms": round(tot["fits_paired"]),
           "in_any_idle_gpu_ms": round(tot["fits_best"]),
           "by_kind": {k: {"transfers": v[0], "moved_ms": round(v[1]), "in_receiver_idle_ms": round(v[2])}
                       for k, v in sorted(by_size.items())}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
