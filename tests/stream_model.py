"""Stream-level model of the executor's enqueue program (runtime.cpp
run_forward / run_backward / run_vocab_fwd / run_vocab_bwd): per rank the
compute stream, one stream per link direction (two-deep receive and send
rings, CUDA events between streams) and the vocab stream; NCCL sends and
receives pair in FIFO order per link, collectives need every rank at the same
op, and optionally the host can only run `Q` ops ahead of completion.
`deadlocks(p, v, m, n, vp)` explores it to a fixpoint.  Used by
tests/test_stream_model.py as a regression check of the protocol (the
executor's device orders come from the planner)."""
from __future__ import annotations

from collections import defaultdict

from paper_2504_14519_b200 import plan as P

KIND = {"F": 0, "B": 1, "W": 2, "BW": 3}


def device_orders(p, v, m, n, vp):
    if vp:
        S = 1024 * n
        r = P.place_vocab(p, v, m, n, True, 1.0 / S, 1.0 / S ** 2, S)
        return [[tuple(x) for x in dev] for dev in r["order"]]
    s = P.gen_slimpipe(p, v, m, n)
    return [[(KIND[s["passes"][i]["kind"]], s["passes"][i]["microbatch"], s["passes"][i]["slice"],
              s["passes"][i]["stage"]) for i in dev] for dev in s["device_order"]]


def build(devs, p, v, vp, depth=2, jit_recv=False):
    nst = p * v
    ops = {}  # (rank, stream) -> list of op dicts
    seqs = {}
    for r, order in enumerate(devs):
        seqs[r] = []
        st = defaultdict(list)
        ev = {}  # event name -> (stream, index) of latest record
        def rec(name, s):
            ev[name] = (s, len(st[s]) - 1)
        def add(s, kind, deps=(), key=None):
            st[s].append({"kind": kind, "deps": [d for d in deps if d is not None], "key": key})
            seqs[r].append((r, s, len(st[s]) - 1))
        def cur(s):
            return (s, len(st[s]) - 1) if st[s] else None
        for x in range(depth):
            for e in ("ain", "out", "gin", "gout"):
                ev[(e, x)] = None
        ain = out = gin = gout = 0
        for (kind, k, i, s) in order:
            if kind == 0:  # F
                if s > 1:
                    b = ain; ain = (ain + 1) % depth
                    add("act_in", "recv", [ev[("ain", b)], cur("act_in")] + ([cur("comp")] if jit_recv else []),
                        ("act", (r - 1) % p, r, k, i, s - 1))
                    add("comp", "wait", [cur("act_in"), cur("comp")])
                    rec(("ain", b), "comp")
                if s < nst:
                    b = out; out = (out + 1) % depth
                    add("comp", "fwd", [ev[("out", b)], cur("comp")])
                    add("act_out", "send", [cur("comp"), cur("act_out")], ("act", r, (r + 1) % p, k, i, s))
                    rec(("out", b), "act_out")
                else:
                    add("comp", "fwd", [cur("comp")])
            elif kind in (4, 5):  # vocab
                nm = ["bcast", "ar1", "ar2"] if kind == 4 else ["reduce"]
                for c in nm:
                    add("vocab", "coll", [cur("comp"), cur("vocab")], (c, k, i))
                    add("comp", "wait", [cur("vocab"), cur("comp")])
            else:  # BW
                gb = None
                if s < nst:
                    gb = gin; gin = (gin + 1) % depth
                    add("grad_in", "recv", [ev[("gin", gb)], cur("grad_in")] + ([cur("comp")] if jit_recv else []),
                        ("grad", (r + 1) % p, r, k, i, s + 1))
                    add("comp", "wait", [cur("grad_in"), cur("comp")])
                    add("comp", "bwd", [cur("comp")])
                else:
                    add("comp", "bwd", [ev[("gout", gout)], cur("comp")])
                if s == 1:
                    if gb is not None:
                        rec(("gin", gb), "comp")
                else:
                    add("grad_out", "send", [cur("comp"), cur("grad_out")], ("grad", r, (r - 1) % p, k, i, s))
                    if gb is not None:
                        rec(("gin", gb), "grad_out")
                    else:
                        rec(("gout", gout), "grad_out"); gout = (gout + 1) % depth
        for s, l in st.items():
            ops[(r, s)] = l
    return ops, seqs

def run(ops, p):
    head = {key: 0 for key in ops}
    done = set()
    def ok_deps(o):
        return all(d is None or (d[0], d[1]) in done for d in o["deps"])
    changed = True
    while changed:
        changed = False
        # local ops
        for (r, s), l in ops.items():
            while head[(r, s)] < len(l):
                o = l[head[(r, s)]]
                if o["kind"] in ("send", "recv", "coll"):
                    break
                deps = [(r,) + d if d is not None else None for d in o["deps"]]
                if not all(d in done for d in deps if d is not None):
                    break
                done.add((r, s, head[(r, s)])); head[(r, s)] += 1; changed = True
        # p2p matching
        for (r, s), l in ops.items():
            if head[(r, s)] >= len(l): continue
            o = l[head[(r, s)]]
            if o["kind"] != "send": continue
            if not all((r,) + d in done for d in o["deps"] if d is not None): continue
            _, src, dst, k, i, stg = o["key"]
            rs = "act_in" if o["key"][0] == "act" else "grad_in"
            l2 = ops.get((dst, rs), [])
            h2 = head.get((dst, rs), 0)
            if h2 < len(l2):
                o2 = l2[h2]
                if o2["key"] == o["key"] and all((dst,) + d in done for d in o2["deps"] if d is not None):
                    done.add((r, s, head[(r, s)])); head[(r, s)] += 1
                    done.add((dst, rs, h2)); head[(dst, rs)] += 1; changed = True
        # collectives
        heads = []
        for r in range(p):
            l = ops.get((r, "vocab"), [])
            h = head.get((r, "vocab"), 0)
            if h >= len(l): break
            o = l[h]
            if not all((r,) + d in done for d in o["deps"] if d is not None): break
            heads.append(o["key"])
        if len(heads) == p and len(set(heads)) == 1:
            for r in range(p):
                done.add((r, "vocab", head[(r, "vocab")])); head[(r, "vocab")] += 1
            changed = True
    stuck = {key: (head[key], ops[key][head[key]]["kind"], ops[key][head[key]]["key"]) for key in ops if head[key] < len(ops[key])}
    return stuck


def run_capped(ops, p, Q, seqs):
    pos = {x: j for r in seqs for j, x in enumerate(seqs[r])}
    head = {key: 0 for key in ops}
    done = set()
    enq = {r: 0 for r in range(p)}
    first_open = {r: 0 for r in range(p)}
    def outstanding(r):
        return sum(1 for x in seqs[r][:enq[r]] if x not in done)
    def is_enq(r, s, i):
        return pos[(r, s, i)] < enq[r]
    def deps_ok(r, o):
        return all((r,) + d in done for d in o["deps"] if d is not None)
    changed = True
    while changed:
        changed = False
        for r in range(p):
            while enq[r] < len(seqs[r]) and outstanding(r) < Q:
                enq[r] += 1; changed = True
        for (r, s), l in ops.items():
            while head[(r, s)] < len(l) and is_enq(r, s, head[(r, s)]):
                o = l[head[(r, s)]]
                if o["kind"] in ("send", "recv", "coll") or not deps_ok(r, o): break
                done.add((r, s, head[(r, s)])); head[(r, s)] += 1; changed = True
        for (r, s), l in ops.items():
            if head[(r, s)] >= len(l) or not is_enq(r, s, head[(r, s)]): continue
            o = l[head[(r, s)]]
            if o["kind"] != "send" or not deps_ok(r, o): continue
            dst = o["key"][2]
            rs = "act_in" if o["key"][0] == "act" else "grad_in"
            l2 = ops.get((dst, rs), []); h2 = head.get((dst, rs), 0)
            if h2 < len(l2) and is_enq(dst, rs, h2) and l2[h2]["key"] == o["key"] and deps_ok(dst, l2[h2]):
                done.add((r, s, head[(r, s)])); head[(r, s)] += 1
                done.add((dst, rs, h2)); head[(dst, rs)] += 1; changed = True
        heads = []
        for r in range(p):
            l = ops.get((r, "vocab"), []); h = head.get((r, "vocab"), 0)
            if h >= len(l) or not is_enq(r, "vocab", h) or not deps_ok(r, l[h]): break
            heads.append(l[h]["key"])
        if len(heads) == p and len(set(heads)) == 1:
            for r in range(p):
                done.add((r, "vocab", head[(r, "vocab")])); head[(r, "vocab")] += 1
            changed = True
    return any(head[k] < len(ops[k]) for k in ops)



def deadlocks(p, v, m, n, vp=False, depth=2, host_queue=None, jit_recv=False) -> bool:
    ops, seqs = build(device_orders(p, v, m, n, vp), p, v, vp, depth, jit_recv)
    if host_queue is None:
        return bool(run(ops, p))
    return run_capped(ops, p, host_queue, seqs)
