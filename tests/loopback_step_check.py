"""One PP > 1 step on ONE GPU through the loopback transport (every rank a
host thread of this process), compared with the float64 oracle
(tests/step_parity.py).  Run as a subprocess by tests/test_loopback_gpu.py,
so a stalled case ends with its own process (and GPU context) instead of
wedging the test session:

    python tests/loopback_step_check.py PP M N EXCHANGE RECOMPUTE [KV_HEADS INTERLEAVE VOCAB_PARALLEL]

(env SP_XMIN / SP_XSKIP=1: the exchange placement filter, slimpipe.h)
Exit code 0 = parity holds; 3 = the step did not finish in time."""
import os

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import sys  # noqa: E402
from pathlib import Path  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import step_parity as SP  # noqa: E402


def main():
    import torch
    from paper_2504_14519_b200.runtime import LoopbackWorld, SlimPipeStep, StepConfig
    pp, m, n = (int(x) for x in sys.argv[1:4])
    x, rc = sys.argv[4], sys.argv[5]
    kv = int(sys.argv[6]) if len(sys.argv) > 6 else 4
    v = int(sys.argv[7]) if len(sys.argv) > 7 else 1
    vp = len(sys.argv) > 8 and sys.argv[8] == "1"
    cfg = StepConfig.c1(pp=pp, microbatches=m, slices=n, layers=2 * pp * v, exchange=x, seq_len=1024 * n,
                        recompute=rc, kv_heads=kv, interleave=v, vocab=1024 if vp else 1000, vocab_parallel=vp,
                        exchange_min_chunks=int(os.environ.get("SP_XMIN", 0)),
                        exchange_skip_last=os.environ.get("SP_XSKIP") == "1")
    world = LoopbackWorld(pp)
    steps = [SlimPipeStep(cfg, r, pp, loopback=world) for r in range(pp)]
    tok, tgt = SP.inputs(cfg)
    torch.cuda.synchronize()
    losses = world.run(lambda r: steps[r].step(tok, tgt, optimizer=False),
                       timeout=float(os.environ.get("SP_STEP_TIMEOUT", 150)), steps=steps)
    if world.errors():
        print("loopback transport saw mismatched message sizes", flush=True)
        sys.exit(1)
    allv = [SP.gather_rank(steps[r], cfg, losses[r]) for r in range(pp)]
    ok, worst, _ = SP.compare(cfg, allv, tok, tgt, log=lambda s: print(s, flush=True))
    xs = [s.exchange_stats() for s in steps]
    if x != "off" and not (sum(s["passes_out"] for s in xs) > 0 and sum(s["bytes_sent"] for s in xs) > 0):
        print("exchange moved no attention work", flush=True)
        ok = False
    for s in steps:
        s.close()
    world.close()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
