"""Multi-GPU (PP = world) sliced-1F1B step parity, launched by torchrun:

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/mp_step_check.py

Each rank runs its stage through the C-ABI executor (NCCL P2P between
stages); parameters and gradients are gathered to rank 0, which runs the
float64 oracle on the same bf16 weights and compares (same tolerances as
tests/test_step_gpu.py).  Exit code 0 = parity holds.
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

NAMES = ["attn_norm", "wqkv", "wo", "mlp_norm", "wgu", "wd"]


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
                        interleave=int(os.environ.get("SP_V", 1)))
    step = SlimPipeStep(cfg, rank, world)
    rng = np.random.default_rng(0)
    tok = rng.integers(0, cfg.vocab, (cfg.microbatches, cfg.seq_len), dtype=np.int32)
    tgt = np.roll(tok, -1, axis=1).astype(np.int32)
    tgt[:, -1] = -1
    loss = step.step(tok, tgt, optimizer=False)
    lps = cfg.layers // world
    mine = {"loss": loss, "params": {}, "grads": {}}
    for l in range(lps):  # lps local layers: v chunks of layers/(pp v)
        for k in NAMES:
            mine["params"][(step.global_layer(l), k)] = step.get_param(l, k)
            mine["grads"][(step.global_layer(l), k)] = step.get_grad(l, k)
    if step.is_first:
        mine["params"][(None, "embedding")] = step.get_param(0, "embedding")
        mine["grads"][(None, "embedding")] = step.get_grad(0, "embedding")
    if step.is_last:
        mine["params"][(None, "final_norm")] = step.get_param(0, "final_norm")
        mine["grads"][(None, "final_norm")] = step.get_grad(0, "final_norm")
    if cfg.vocab_parallel:  # every stage holds a vocabulary shard of the head
        mine["head_shard"] = (step.get_param(0, "head"), step.get_grad(0, "head"))
    elif step.is_last:
        mine["params"][(None, "head")] = step.get_param(0, "head")
        mine["grads"][(None, "head")] = step.get_grad(0, "head")
    mem = step.memory()
    mine["mem"] = mem
    mine["x"] = step.exchange_stats()
    allv = [None] * world
    dist.all_gather_object(allv, mine)
    ok = True
    if rank == 0:
        import model_oracle as MO
        P, G = {}, {}
        for d in allv:
            P.update(d["params"])
            G.update(d["grads"])
        if cfg.vocab_parallel:
            P[(None, "head")] = np.concatenate([d["head_shard"][0] for d in allv], axis=0)
            G[(None, "head")] = np.concatenate([d["head_shard"][1] for d in allv], axis=0)
        rnd = lambda x: torch.from_numpy(x).bfloat16().double().numpy()
        W = {k: [rnd(P[(l, k)]) for l in range(cfg.layers)] for k in NAMES}
        for k in ("embedding", "final_norm", "head"):
            W[k] = rnd(P[(None, k)])
        ref_loss, ref_g = MO.Model(W, cfg.heads, cfg.kv_heads, cfg.rope_theta, cfg.norm_eps).step(tok, tgt, n)
        gpu_loss = allv[-1]["loss"]
        print(f"pp={world} v={cfg.interleave} m={m} n={n} exchange={xmode} vocab_parallel={cfg.vocab_parallel} "
              f"loss gpu {gpu_loss:.6f} oracle {ref_loss:.6f}")
        xs = [d["x"] for d in allv]
        print("exchange stats per rank:", xs)
        if xmode != "off":
            ok &= sum(x["passes_out"] for x in xs) > 0 and sum(x["bytes_sent"] for x in xs) > 0
        ok &= abs(gpu_loss - ref_loss) / abs(ref_loss) < 1e-2
        worst = 0.0
        for (l, k), g in G.items():
            r = ref_g[k][l] if l is not None else ref_g[k]
            e = float(np.max(np.abs(g - r)) / max(1e-30, np.max(np.abs(r))))
            worst = max(worst, e)
            if e > 5e-2:
                print("grad mismatch", l, k, e)
                ok = False
        for r_, d in enumerate(allv):
            mm = d["mem"]
            expect = n + 2 * (world - 1 - r_) if m * n >= n + 2 * (world - 1) and cfg.interleave == 1 else None
            print(f"rank {r_}: slots {mm['slots']} high-water {mm['slots_high_water']} ledger {mm['ledger_peak_units']}"
                  f" (n+2(p-d) = {expect})")
            ok &= mm["slots_high_water"] == mm["ledger_peak_units"]
        print("worst grad err", worst, "PASS" if ok else "FAIL")
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(flag, 0)
    step.close()
    dist.destroy_process_group()
    sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
