"""Timed version of the stream-level model (tests/stream_model.py, which
reproduces the measured VP+exchange stall state exactly): every compute op
gets a duration taken from a MEASURED exchange-off step (per-pass spans of
its Gantt; per-chunk attention cost from a per-stage line fit), transfers
take bytes / link rate, and a GPU's serve compute (high-priority stream)
pre-empts its own pass while it runs.  It predicts the step time of the
executor with the reference plan's exchange — unfiltered, with the placement
filter, and with per-sender serve lanes (a design) — from the
off measurement alone, so its predictions for the built variants can be
checked against their measured lines.

    python scripts/exchange_timed_model.py GANTT_OFF.json P M N SEQ HIDDEN KV_DIM [--layers L] [--gbs 500]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import stream_model as SM  # noqa: E402

KCODE = {"F": 0, "BW": 3}


def measured(path):
    g = json.loads(Path(path).read_text())
    dur = {}
    for row in g["rows"]:
        for x in row:
            dur[(KCODE[x["kind"]], x["microbatch"], x["slice"], x["stage"])] = x["end"] - x["start"]
    fits = {}
    for (kd, _, i, s), d in dur.items():
        fits.setdefault((kd, s), []).append((i, d))
    per_chunk = {}
    for key, pts in fits.items():
        x, y = np.array(pts, float).T
        b, a = np.polyfit(x, y, 1)
        per_chunk[key] = max(0.0, float(b))  # ms of attention per attended chunk (all layers of the pass)
    return g["makespan"], dur, per_chunk


def idle_placed(p, m, n, mode, gantt, per_chunk, min_fill=0.5):
    """The plan's transfers kept only where the receiving GPU is idle, in the
    measured off step, for at least min_fill of the moved attention inside
    the sending pass's window (a placement by measured idle time; not built)."""
    from paper_2504_14519_b200 import plan as P
    g = json.loads(Path(gantt).read_text())
    rows = [sorted(r, key=lambda x: x["start"]) for r in g["rows"]]
    span = {(KCODE[x["kind"]], x["microbatch"], x["slice"], x["stage"]): (x["start"], x["end"]) for r in rows for x in r}
    passes = P.gen_slimpipe(p, 1, m, n)["passes"]
    key = {q["id"]: (KCODE[q["kind"]], q["microbatch"], q["slice"], q["stage"]) for q in passes}

    def idle_in(row, a, b):
        return (b - a) - sum(max(0.0, min(b, x["end"]) - max(a, x["start"])) for x in row)

    keep = set()
    for t in P.apply_exchange(p, 1, m, n, mode)["ticks"]:
        pid = {d: q for d, _, q in t["in"]}
        for tr in t["plan"]["transfers"]:
            sp, dp = pid[tr["src"]], pid[tr["dst"]]
            s0, s1 = span[key[sp]]
            work = per_chunk[(key[sp][0], key[sp][3])] * len(tr["chunks"])
            if idle_in(rows[tr["dst"] - 1], s0, s1) >= min_fill * work:
                keep.add((sp, tr["dst"] - 1, tuple(tr["chunks"])))
                keep.add(("in", dp, tr["src"] - 1, tuple(tr["chunks"])))
    return keep


def simulate(p, m, n, mode, dur, per_chunk, layers, sizes, gbs, min_chunks=0, skip_last=False, lanes=False,
             gated=False, keep=None):
    """gated: a communication kernel (stage or exchange, normal-priority stream)
    is dispatched only once the rank's compute stream is not inside an
    attention kernel (K1/K2: one launch per layer, tens of ms) — the
    equal-priority dispatch order of the hardware; False: communication
    streams of high priority (dispatched at once)."""
    devs, pids, xw = SM.exchange_program(p, m, n, mode if mode != "off" else "on", min_chunks, skip_last)
    if mode == "off":
        xw = [{} for _ in range(p)]
    elif keep is not None:  # placement by measured idle time
        for r in range(p):
            for pid, px in list(xw[r].items()):
                px = dict(px)
                px["out"] = [o for o in px["out"] if (pid, o["peer"], tuple(o["chunks"])) in keep]
                px["in"] = [i for i in px["in"] if ("in", pid, i["peer"], tuple(i["chunks"])) in keep]
                xw[r][pid] = px
    ops, _ = SM.build(devs, p, 1, False, 2, True, pids, xw, layers, True, lanes)
    Ls, qd, kvd = sizes

    def attn_part(o):
        kd, _, i, stg = o["at"]
        moved = o["key"][1] if len(o["key"]) > 1 else 0
        whole = dur[o["at"]] / layers
        attn = min(whole * 0.95, per_chunk[(kd, stg)] * i / layers)
        return whole - attn, max(0.0, attn - per_chunk[(kd, stg)] * moved / layers)

    def duration(r, o):
        k = o["kind"]
        if k in ("fwd", "bwd") and o["key"] and o["key"][0] == "attn":
            lin, attn = attn_part(o)
            return lin + attn
        if k == "xcomp":
            _, c, src, _, nch = o["key"]
            return per_chunk[(0 if c == 0 else 3, src + 1)] * nch / layers
        return 0.0

    def xfer_ms(o):
        tag, c = o["key"][0], o["key"][1]
        if tag in ("act", "grad"):
            return Ls * qd * 2 / (gbs * 1e6)
        return 0.0  # priced on the send side below

    # per-op durations
    D = {(r, s, j): duration(r, o) for (r, s), l in ops.items() for j, o in enumerate(l)}
    ATT = {(r, s, j): attn_part(o)[1] for (r, s), l in ops.items() for j, o in enumerate(l)
           if o["kind"] in ("fwd", "bwd") and o["key"] and o["key"][0] == "attn"}

    def in_attention(r):
        rem = running.get((r, "comp"))
        return rem is not None and rem <= ATT.get((r, "comp", head[(r, "comp")]), 0.0) + 1e-9
    head = {key: 0 for key in ops}
    running = {}  # (r, s) -> remaining ms  (for p2p, both ends hold the same entry)
    partner = {}
    done = set()
    t = 0.0

    def deps_ok(r, o):
        return all((r,) + d in done for d in o["deps"] if d is not None)

    def xbytes(o, nch_of):
        tag, c = o["key"][0], o["key"][1]
        if tag == "xreq":
            return Ls * qd * 2 * (1 if c == 0 else 2) + nch_of * 2 * Ls * kvd * 2
        return Ls * qd * (2 if c == 0 else 4) + (0 if c == 0 else nch_of * 2 * Ls * kvd * 4)

    # chunks per transfer: from the serve compute that follows each request on the receiver
    nch = {}
    for (r, s), l in ops.items():
        for j, o in enumerate(l):
            if o["kind"] == "xcomp":
                _, c, src, dst, n_ = o["key"]
                nch.setdefault((c, src, dst), []).append(n_)
    seen = {}

    def chunks_for(o):
        _, c, a, b, ordinal = o["key"]
        src, dst = (a, b) if o["key"][0] == "xreq" else (b, a)
        lst = nch.get((c, src, dst), [])
        return lst[ordinal % len(lst)] if lst else 0

    while True:
        progress = True
        while progress:
            progress = False
            for (r, s), l in ops.items():
                h = head[(r, s)]
                if h >= len(l) or (r, s) in running:
                    continue
                o = l[h]
                if o["kind"] in ("send", "recv", "xsend", "xrecv", "coll") or not deps_ok(r, o):
                    continue
                d = D[(r, s, h)]
                if d <= 0:
                    done.add((r, s, h)); head[(r, s)] += 1; progress = True
                else:
                    running[(r, s)] = d
            for (r, s), l in ops.items():
                h = head[(r, s)]
                if h >= len(l) or (r, s) in running:
                    continue
                o = l[h]
                if o["kind"] not in ("send", "xsend") or not deps_ok(r, o):
                    continue
                if o["kind"] == "send":
                    dst = o["key"][2]
                    ts = "act_in" if o["key"][0] == "act" else "grad_in"
                    ms = xfer_ms(o)
                else:
                    dst, ts = o["to"]
                    ms = xbytes(o, chunks_for(o)) / (gbs * 1e6)
                if gated and o["kind"] == "xsend" and (in_attention(r) or in_attention(dst)):
                    continue  # stage messages: their dispatch delays are inside the measured off spans
                l2, h2 = ops.get((dst, ts), []), head.get((dst, ts), 0)
                if h2 < len(l2) and (dst, ts) not in running and l2[h2]["key"] == o["key"] and deps_ok(dst, l2[h2]):
                    running[(r, s)] = ms
                    running[(dst, ts)] = ms
                    partner[(r, s)] = (dst, ts)
                    partner[(dst, ts)] = (r, s)
                    progress = True
        if not running:
            break
        # rates: a rank's serve compute pre-empts its compute stream
        rate = {}
        for (r, s) in running:
            if s == "comp":
                busy_rx = any(rr == r and ss.startswith("rx") for (rr, ss) in running)
                rate[(r, s)] = 0.0 if busy_rx else 1.0
            elif s.startswith("rx"):
                nrx = sum(1 for (rr, ss) in running if rr == r and ss.startswith("rx"))
                rate[(r, s)] = 1.0 / nrx
            else:
                rate[(r, s)] = 1.0
        dt = min(rem / rate[k] for k, rem in running.items() if rate[k] > 0)
        t += dt
        finished = []
        for k in list(running):
            running[k] -= dt * rate[k]
            if running[k] <= 1e-9:
                finished.append(k)
        for k in finished:
            if k in running:
                del running[k]
                r, s = k
                done.add((r, s, head[k])); head[k] += 1
                if k in partner:
                    q = partner.pop(k)
                    partner.pop(q, None)
                    if q in running:
                        del running[q]
                        done.add((q[0], q[1], head[q])); head[q] += 1
    stuck = any(head[k] < len(ops[k]) for k in ops)
    return t, stuck


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("gantt")
    for a in ("p", "m", "n", "seq", "hidden", "kv_dim"):
        ap.add_argument(a, type=int)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--gbs", type=float, default=500.0)
    ap.add_argument("--mode", default="early")
    ap.add_argument("--min-chunks", type=int, default=2)
    a = ap.parse_args()
    mk, dur, per_chunk = measured(a.gantt)
    sizes = (a.seq // a.n, a.hidden, a.kv_dim)
    tok = a.m * a.seq
    out = {"measured_off_makespan_ms": mk}
    keep = idle_placed(a.p, a.m, a.n, a.mode, a.gantt, per_chunk)
    for gated in (True, False):
        tag = "gated" if gated else "prompt"
        for name, kw in [("off", dict(mode="off")), ("plan", dict(mode=a.mode)),
                         ("idle_placed", dict(mode=a.mode, keep=keep)),
                         ("idle_placed_lanes", dict(mode=a.mode, keep=keep, lanes=True)),
                         ("filtered", dict(mode=a.mode, min_chunks=a.min_chunks, skip_last=True)),
                         ("plan_lanes", dict(mode=a.mode, lanes=True)),
                         ("filtered_lanes", dict(mode=a.mode, min_chunks=a.min_chunks, skip_last=True, lanes=True))]:
            ms, stuck = simulate(a.p, a.m, a.n, dur=dur, per_chunk=per_chunk, layers=a.layers, sizes=sizes,
                                 gbs=a.gbs, gated=gated, **kw)
            out[f"{tag}/{name}"] = {"makespan_ms": round(ms, 1), "tokens_per_s": round(tok / (ms / 1e3)),
                                    "stuck": stuck}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
