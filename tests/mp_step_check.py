"""Multi-GPU (PP = world) sliced-1F1B step parity, launched by torchrun:

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/mp_step_check.py

Each rank runs its stage through the C-ABI executor (NCCL P2P between
stages); parameters and gradients are gathered to rank 0, which runs the
float64 oracle on the same bf16 weights and compares (same tolerances as
tests/test_step_gpu.py).  Exit code 0 = parity holds.
"""
import os

# one hardware work queue per CUDA stream (the executor runs up to ten per
# rank; shared queues let a waiting stream stall unrelated ones) — before the
# CUDA context exists
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT / "tests"))

import step_parity as SP  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0))))
    from paper_2504_14519_b200.runtime import SlimPipeStep, StepConfig
    m = int(os.environ.get("SP_M", 2))
    n = int(os.environ.get("SP_N", 4))
    xmode = os.environ.get("SP_X", "off")
    vp = os.environ.get("SP_VP") == "1"
    cfg = StepConfig.c1(pp=world, microbatches=m, slices=n, layers=2 * world, exchange=xmode,
                        vocab=1024 if vp else 1000,  # vocab shards must be a multiple of 4 wide
                        seq_len=1024 * n, recompute=os.environ.get("SP_RC", "selective"),
                        kv_heads=int(os.environ.get("SP_KV", 4)), vocab_parallel=vp,
                        interleave=int(os.environ.get("SP_V", 1)), offload=os.environ.get("SP_OFFLOAD") == "1",
                        exchange_min_chunks=int(os.environ.get("SP_XMIN", 0)),
                        exchange_skip_last=os.environ.get("SP_XSKIP") == "1")
    step = SlimPipeStep(cfg, rank, world)
    tok, tgt = SP.inputs(cfg)
    # the step on a watched thread: a stall reports where this rank stands
    import threading
    import time
    from paper_2504_14519_b200.runtime import _lib
    box = {}
    th = threading.Thread(target=lambda: box.setdefault("loss", step.step(tok, tgt, optimizer=False)), daemon=True)
    th.start()
    th.join(float(os.environ.get("SP_STEP_TIMEOUT", 240)))
    if th.is_alive():
        print(f"rank {rank}: step stalled; host enqueuing pass #{_lib().sp_runtime_enqueue_position(step._h)}, "
              f"device at {step.progress()}", flush=True)
        time.sleep(2)
        os._exit(3)
    loss = box["loss"]
    mine = SP.gather_rank(step, cfg, loss)
    allv = [None] * world
    dist.all_gather_object(allv, mine)
    ok = True
    if rank == 0:
        ok, _, _ = SP.compare(cfg, allv, tok, tgt)
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(flag, 0)
    step.close()
    dist.destroy_process_group()
    sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
