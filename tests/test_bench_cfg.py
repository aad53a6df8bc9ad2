"""bench.py's configuration layer on the CPU: the flags reach StepConfig (and
through it sp_model_config), the workload string names what runs, and the
combinations the runtime rejects are not produced by the defaults."""
from __future__ import annotations

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def _cfg(argv, world):
    import bench
    old = sys.argv
    sys.argv = ["bench.py", *argv]
    try:
        args = bench.parse()
    finally:
        sys.argv = old
    return bench, bench.make_cfg(args, world), args


def test_default_is_the_c2_workload_at_pp_n():
    bench, cfg, _ = _cfg([], 1)
    assert (cfg.layers, cfg.hidden, cfg.heads, cfg.seq_len, cfg.slices, cfg.microbatches) == (8, 4096, 32, 131072, 8, 4)
    assert cfg.pp == 1 and cfg.exchange == "off" and not cfg.vocab_parallel and cfg.interleave == 1
    assert not cfg.offload and not cfg.dkv_bf16 and cfg.exchange_min_chunks == 0 and not cfg.exchange_skip_last
    name = bench.workload_name(cfg, "c2")
    assert "PP=1" in name and "exchange=off" in name and "128K" in name


def test_flags_reach_the_step_config():
    bench, cfg, _ = _cfg(["--exchange", "early", "--exchange-min-chunks", "3", "--exchange-skip-last",
                          "--dkv-bf16", "--offload"], 4)
    assert cfg.pp == 4 and cfg.exchange == "early" and cfg.exchange_min_chunks == 3 and cfg.exchange_skip_last
    assert cfg.dkv_bf16 and cfg.offload
    c = cfg.to_c(0)
    assert (c.exchange_mode, c.exchange_min_chunks, c.exchange_skip_last, c.dkv_bf16, c.offload) == (2, 3, 1, 1, 1)
    name = bench.workload_name(cfg, "c2")
    assert "min 3 chunks" in name and "last stage" in name and "bf16 dK/dV" in name


def test_single_gpu_drops_multi_stage_options():
    _, cfg, _ = _cfg(["--vocab-parallel", "--interleave", "2"], 1)
    assert not cfg.vocab_parallel and cfg.interleave == 1


@pytest.mark.parametrize("model,layers,seq,world", [("c3", 8, 262144, 4), ("c4", 2, 1 << 20, 1)])
def test_model_presets(model, layers, seq, world):
    _, cfg, _ = _cfg(["--model", model], world)
    assert (cfg.layers, cfg.seq_len, cfg.pp) == (layers, seq, world)
    assert cfg.layers % cfg.pp == 0
