"""K2 A/B: time backward kernel variants on the c2 representative slices,
one process per variant (the library read SP_BWD_VARIANT once while the
variants were compiled in; the winner is now the only build — see
profiles/r02_k2_ab.json for the measured variants), and check they agree.
Writes gpurun_out/k2_ab.json."""
import json
import os
import subprocess
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
HEADS, D = 32, 128
SHAPES = [(16384, 4), (16384, 8), (8192, 16)]


def child():
    from paper_2504_14519_b200 import ops
    out = {}
    for L, n in SHAPES:
        g = torch.Generator(device="cuda").manual_seed(7)
        mk = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16, generator=g)
        q, kp, vp, do = mk(L, HEADS * D), mk(n * L, HEADS * D), mk(n * L, HEADS * D), mk(L, HEADS * D)
        rows = [c * L for c in range(n)]
        o, lse = ops.attn_fwd(q, kp, vp, rows, L, HEADS, HEADS, True)
        dq = torch.zeros(L, HEADS * D, device="cuda")
        dk = torch.zeros(n * L, HEADS * D, device="cuda")
        dv = torch.zeros_like(dk)
        ws = torch.empty(2 * HEADS * L, device="cuda")
        run = lambda: ops.attn_bwd(q, kp, vp, rows, L, HEADS, HEADS, True, o, lse, do, dq, dk, dv, rows, ws)
        run()
        torch.cuda.synchronize()
        ck = [float(dq.double().sum()), float(dk.double().sum()), float(dv.double().norm())]
        for _ in range(2):
            run()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        it = 5
        s.record()
        for _ in range(it):
            run()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / it
        fl = 2.5 * 4.0 * D * L * ((n - 1) * L + (L + 1) / 2) * HEADS
        out[f"{L}x{n}"] = {"ms": ms, "tflops": fl / ms / 1e9, "check": ck}
    print(json.dumps(out))


if __name__ == "__main__":
    if len(sys.argv) > 1:
        child()
        sys.exit(0)
    res = {}
    for v in os.environ.get("VARIANTS", "0 1 2").split():
        var = os.environ.get("VARIANT_VAR", "SP_BWD_VARIANT")
        r = subprocess.run([sys.executable, __file__, "child"], env=dict(os.environ, **{var: v}),
                           capture_output=True, text=True, timeout=600)
        line = [x for x in r.stdout.splitlines() if x.startswith("{")]
        res[v] = json.loads(line[-1]) if line else {"error": r.stderr[-2000:]}
        print(v, json.dumps(res[v]), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(res, open("gpurun_out/k2_ab.json", "w"), indent=1)
