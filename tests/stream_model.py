"""Stream-level model of the executor's enqueue program (runtime.cpp
run_forward / run_backward / run_vocab_fwd / run_vocab_bwd): per rank the
compute stream, one stream per link direction (two-deep receive and send
rings, CUDA events between streams) and the vocab stream; NCCL sends and
receives pair in FIFO order per link, collectives need every rank at the same
op, and optionally the host can only run `Q` ops ahead of completion.
With the exchange, each class has a request/serve stream cx<c> and a serve
compute stream rx<c>; its sends and receives pair FIFO per (class, sender,
receiver) at the heads of the two ranks' cx<c>, and the transfer lists are
the executor's own (sp_exchange_passes_json).
`deadlocks(p, v, m, n, vp)` / `exchange_deadlocks(...)` explore it to a fixpoint.  Used by
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


def build(devs, p, v, vp, depth=2, jit_recv=False, pids=None, xw=None, layers=2, serve_jit=True, lanes=False):
    """pids[r][j]: pass id of devs[r][j] (F/BW; None for vocab passes); xw[r]:
    the executor's exchange wiring of rank r ({pass id: px}, from
    sp_exchange_passes_json) — then every layer of a shipping pass sends its
    requests on the class stream cx<c> and waits there for the partials, and a
    serving pass posts its serves (recv request, compute on rx<c>, send the
    partial) at its start, as runtime.cpp attention_forward / layer_backward /
    post_remote do (selective recompute).  lanes=True: each sender's serves on
    their own stream pair cx<c>s<src> / rx<c>s<src> (a design, not the
    executor: one communicator per sending stage)."""
    nst = p * v
    ops = {}  # (rank, stream) -> list of op dicts
    seqs = {}
    req = defaultdict(int)  # (cls, src, dst) -> requests enqueued by the sender so far
    res = defaultdict(int)
    srv_req = defaultdict(int)  # same counters on the serving side (FIFO matching per pair)
    srv_res = defaultdict(int)
    for r, order in enumerate(devs):
        seqs[r] = []
        st = defaultdict(list)
        ev = {}  # event name -> (stream, index) of latest record
        def rec(name, s):
            ev[name] = (s, len(st[s]) - 1)
        at = [None]  # the pass being enqueued (diagnostics: where a stream is stuck)

        def add(s, kind, deps=(), key=None):
            st[s].append({"kind": kind, "deps": [d for d in deps if d is not None], "key": key, "at": at[0]})
            seqs[r].append((r, s, len(st[s]) - 1))
        def cur(s):
            return (s, len(st[s]) - 1) if st[s] else None
        for x in range(depth):
            for e in ("ain", "out", "gin", "gout"):
                ev[(e, x)] = None
        ain = out = gin = gout = 0

        def lane(c, src):
            return (f"cx{c}s{src}", f"rx{c}s{src}") if lanes else (f"cx{c}", f"rx{c}")

        def serve(px):  # post_remote
            c = px["cls"]
            if serve_jit:
                for cx in {lane(c, t["peer"])[0] for t in px["in"]}:
                    add(cx, "wait", [cur("comp"), cur(cx)])
            for _ in range(layers):
                for t in px["in"]:
                    src = t["peer"]
                    cx, rx = lane(c, src)
                    add(cx, "xrecv", [cur(cx)], ("xreq", c, src, r, srv_req[(c, src, r)]))
                    srv_req[(c, src, r)] += 1
                    add(rx, "xcomp", [cur(cx), cur(rx)], ("xwork", c, src, r, len(t["chunks"])))
                    add(cx, "xsend", [cur(rx), cur(cx)], ("xres", c, r, src, srv_res[(c, r, src)]))
                    st[cx][-1]["to"] = (src, f"cx{c}")
                    srv_res[(c, r, src)] += 1

        def attention(px, step):  # attention_forward / the K2 part of layer_backward
            if not px or not px["out"]:
                add("comp", step, [cur("comp")], ("attn",))
                return
            c = px["cls"]
            cx = f"cx{c}"
            add(cx, "wait", [cur("comp"), cur(cx)])
            for o in px["out"]:
                add(cx, "xsend", [cur(cx)], ("xreq", c, r, o["peer"], req[(c, r, o["peer"])]))
                st[cx][-1]["to"] = (o["peer"], lane(c, r)[0])
                req[(c, r, o["peer"])] += 1
            add("comp", step, [cur("comp")], ("attn", sum(len(o["chunks"]) for o in px["out"])))
            for o in px["out"]:
                add(cx, "xrecv", [cur(cx)], ("xres", c, o["peer"], r, res[(c, o["peer"], r)]))
                res[(c, o["peer"], r)] += 1
            add("comp", "wait", [cur(cx), cur("comp")])

        for j, (kind, k, i, s) in enumerate(order):
            at[0] = (kind, k, i, s)
            px = xw[r].get(pids[r][j]) if xw is not None and pids[r][j] is not None else None
            if px and px["in"]:
                serve(px)
            if kind == 0:  # F
                if s > 1:
                    b = ain; ain = (ain + 1) % depth
                    add("act_in", "recv", [ev[("ain", b)], cur("act_in")] + ([cur("comp")] if jit_recv else []),
                        ("act", (r - 1) % p, r, k, i, s - 1))
                    add("comp", "wait", [cur("act_in"), cur("comp")])
                    rec(("ain", b), "comp")
                if xw is not None:
                    for _ in range(layers):
                        attention(px, "fwd")
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
                if xw is not None:
                    for _ in range(layers):
                        attention(px, "bwd")
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
                if o["kind"] in ("send", "recv", "coll", "xsend", "xrecv"):
                    break
                deps = [(r,) + d if d is not None else None for d in o["deps"]]
                if not all(d in done for d in deps if d is not None):
                    break
                done.add((r, s, head[(r, s)])); head[(r, s)] += 1; changed = True
        # exchange p2p: a send at the head of one rank's class stream meets
        # the matching receive at the head of the peer's
        for (r, s), l in ops.items():
            if not s.startswith("cx") or head[(r, s)] >= len(l):
                continue
            o = l[head[(r, s)]]
            if o["kind"] != "xsend" or not all((r,) + d in done for d in o["deps"] if d is not None):
                continue
            dst, ts = o["to"]
            l2, h2 = ops.get((dst, ts), []), head.get((dst, ts), 0)
            if h2 < len(l2):
                o2 = l2[h2]
                if o2["kind"] == "xrecv" and o2["key"] == o["key"] and \
                        all((dst,) + d in done for d in o2["deps"] if d is not None):
                    done.add((r, s, head[(r, s)])); head[(r, s)] += 1
                    done.add((dst, ts, h2)); head[(dst, ts)] += 1; changed = True
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
    stuck = {key: (head[key], ops[key][head[key]]["kind"], ops[key][head[key]]["key"], ops[key][head[key]].get("at"))
             for key in ops if head[key] < len(ops[key])}
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


def exchange_program(p, m, n, mode, min_chunks=0, skip_last=False, vp=False):
    """Device orders, pass ids and the executor's exchange wiring (v = 1)."""
    sch = P.gen_slimpipe(p, 1, m, n)
    pid_of = {(KIND[q["kind"]], q["microbatch"], q["slice"], q["stage"]): q["id"] for q in sch["passes"]}
    devs = device_orders(p, 1, m, n, vp)
    pids = [[pid_of.get(tuple(e)) for e in dev] for dev in devs]
    xw = [{px["pass"]: px for px in P.exchange_passes(p, m, n, mode, r, min_chunks, skip_last)} for r in range(p)]
    return devs, pids, xw


def exchange_deadlocks(p, m, n, mode, min_chunks=0, skip_last=False, vp=False, serve_jit=True, jit_recv=True,
                       layers=2, lanes=False) -> dict:
    devs, pids, xw = exchange_program(p, m, n, mode, min_chunks, skip_last, vp)
    ops, _ = build(devs, p, 1, vp, 2, jit_recv, pids, xw, layers, serve_jit, lanes)
    return run(ops, p)
