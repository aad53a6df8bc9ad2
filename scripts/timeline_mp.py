"""Per-rank pass timelines of one step (torchrun, N GPUs) for exchange on/off.

    torchrun --nproc-per-node 4 scripts/timeline_mp.py --exchange early
Prints per pass (rank, kind, k, i, start_ms, end_ms) relative to a barrier-
aligned step start, plus per-rank busy / idle and the bubble fraction.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2504_14519_b200 import plan as PL  # noqa: E402
from paper_2504_14519_b200.runtime import SlimPipeStep, StepConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--exchange", default="off")
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--seq-len", type=int, default=65536)
ap.add_argument("--slices", type=int, default=8)
ap.add_argument("--microbatches", type=int, default=4)
ap.add_argument("--out", default="gpurun_out/timeline.json")
a = ap.parse_args()
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0))))
cfg = StepConfig.c2(layers=a.layers, seq_len=a.seq_len, slices=a.slices, microbatches=a.microbatches, pp=world,
                    exchange=a.exchange)
step = SlimPipeStep(cfg, rank, world)
rng = np.random.default_rng(0)
tok = torch.from_numpy(rng.integers(0, cfg.vocab, (cfg.microbatches, cfg.seq_len), dtype=np.int32)).cuda()
for _ in range(2):
    step.step_async(tok.data_ptr(), tok.data_ptr())
step.sync()
dist.barrier()
torch.cuda.synchronize()
step.step_async(tok.data_ptr(), tok.data_ptr())
step.sync()
ms, passes = step.timeline()
sched = PL.gen_slimpipe(world, 1, cfg.microbatches, cfg.slices)
mine = [(rank, sched["passes"][pid]["kind"], sched["passes"][pid]["microbatch"], sched["passes"][pid]["slice"], s, e)
        for pid, s, e in passes]
allv = [None] * world
dist.all_gather_object(allv, {"ms": ms, "passes": mine, "x": step.exchange_stats()})
if rank == 0:
    span = max(v["ms"] for v in allv)
    busy = [sum(e - s for *_, s, e in v["passes"]) for v in allv]
    print(f"exchange={a.exchange} step {span:.1f} ms  busy per rank {[round(b) for b in busy]}  "
          f"bubble {(world * span - sum(busy)) / sum(busy):.3f}  x={[v['x'] for v in allv]}")
    for v in allv:
        line = " ".join(f"{k}{mb}.{i}:{s:.0f}-{e:.0f}" for (_, k, mb, i, s, e) in v["passes"][:40])
        print(f"r{v['passes'][0][0]} {line}")
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(allv, open(a.out.replace(".json", f"_{a.exchange}.json"), "w"))
step.close()
dist.destroy_process_group()
