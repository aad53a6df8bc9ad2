"""End-to-end parity of one sliced-1F1B training step (tiny config c1) on the
GPU against the float64 oracle (oracle/model_oracle.py, whose attention is the
C restatement of the reference chunk_attention).

Weights are read back from the device and rounded to bf16 (the GPU computes
with bf16 weights and bf16 activations, fp32 accumulation), so the oracle sees
exactly the same parameters.  Tolerances: loss rel 1e-2;
gradients max|gpu - oracle| <= 4e-2 * max|oracle| per tensor (bf16 activations
through the whole stack).
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))
import model_oracle as MO  # noqa: E402

pytestmark = pytest.mark.gpu
LOSS_TOL = 1e-2
GRAD_TOL = 4e-2  # measured worst 2.8 % (attn_norm, PP=4 v=2 full); typical 0.7-1.2 %
NAMES = ["attn_norm", "wqkv", "wo", "mlp_norm", "wgu", "wd"]


def _bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).bfloat16().double().numpy()


def _nerr(a, b):
    return float(np.max(np.abs(a - b)) / max(1e-30, np.max(np.abs(b))))


def _data(cfg, seed=0):
    rng = np.random.default_rng(seed)
    tok = rng.integers(0, cfg.vocab, size=(cfg.microbatches, cfg.seq_len), dtype=np.int32)
    tgt = np.roll(tok, -1, axis=1).astype(np.int32)
    tgt[:, -1] = -1
    return tok, tgt


def _pull(step, cfg):
    W = {k: [] for k in NAMES}
    for l in range(cfg.layers):
        for k in NAMES:
            W[k].append(_bf16(step.get_param(l, k)))
    for k in ("embedding", "final_norm", "head"):
        W[k] = _bf16(step.get_param(0, k))
    return W


@pytest.mark.parametrize("m,n,rc,shape", [(2, 4, "selective", {}), (1, 2, "selective", {}), (2, 4, "full", {}),
                                          # GQA 4:2 on the d=64 kernels, and d=128 (production K1/K2) with GQA
                                          (2, 4, "selective", {"kv_heads": 2}),
                                          (2, 4, "selective", {"hidden": 512, "kv_heads": 2, "ffn_hidden": 1024}),
                                          (1, 4, "full", {"hidden": 512, "kv_heads": 4, "ffn_hidden": 1024}),
                                          # activation offload (stage input + O/LSE via pinned host memory)
                                          (2, 4, "selective", {"offload": True}),
                                          (2, 4, "full", {"offload": True, "hidden": 512, "ffn_hidden": 1024}),
                                          # bf16 dK/dV accumulators (d=64 and d=128 kernels)
                                          (2, 4, "selective", {"dkv_bf16": True}),
                                          (2, 4, "selective", {"dkv_bf16": True, "hidden": 512, "kv_heads": 2,
                                                               "ffn_hidden": 1024})],
                         ids=["base", "m1n2", "full", "gqa", "d128-gqa", "d128-full", "offload", "offload-d128-full",
                              "dkv-bf16", "dkv-bf16-d128-gqa"])
def test_c1_step_matches_oracle(m, n, rc, shape):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_14519_b200.runtime import SlimPipeStep, StepConfig
    cfg = StepConfig.c1(microbatches=m, slices=n, recompute=rc, **shape)
    step = SlimPipeStep(cfg, rank=0, world=1)
    tok, tgt = _data(cfg)
    loss = step.step(tok, tgt, optimizer=False)
    W = _pull(step, cfg)
    ref_loss, ref_g = MO.Model(W, cfg.heads, cfg.kv_heads, cfg.rope_theta, cfg.norm_eps).step(tok, tgt, n)
    assert abs(loss - ref_loss) / abs(ref_loss) < LOSS_TOL, (loss, ref_loss)
    worst = {}
    for l in range(cfg.layers):
        for k in NAMES:
            worst[f"{k}{l}"] = _nerr(step.get_grad(l, k), ref_g[k][l])
    for k in ("embedding", "final_norm", "head"):
        worst[k] = _nerr(step.get_grad(0, k), ref_g[k])
    bad = {k: v for k, v in worst.items() if v > GRAD_TOL}
    assert not bad, (bad, worst)
    mem = step.memory()
    assert mem["slots_high_water"] == mem["ledger_peak_units"] == mem["slots"]
    step.close()


def test_c1_optimizer_step_changes_weights_and_loss_is_stable():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_14519_b200.runtime import SlimPipeStep, StepConfig
    cfg = StepConfig.c1(lr=1e-3)
    step = SlimPipeStep(cfg, rank=0, world=1)
    tok, tgt = _data(cfg, 1)
    w0 = step.get_param(0, "wqkv")
    l0 = step.step(tok, tgt)
    w1 = step.get_param(0, "wqkv")
    l1 = step.step(tok, tgt)
    assert np.max(np.abs(w1 - w0)) > 0
    assert np.isfinite(l0) and np.isfinite(l1) and l1 < l0  # same batch: loss must drop
    step.close()
