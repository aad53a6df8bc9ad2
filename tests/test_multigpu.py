"""PP > 1 on real GPUs: runs tests/mp_step_check.py under torchrun when at
least 2 GPUs are visible (gpurun --gpus 2|4)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("pp,m,n,x,rc", [(2, 2, 4, "off", "selective"), (2, 1, 2, "off", "full"),
                                         (2, 2, 4, "on", "selective"), (2, 2, 4, "on", "full"),
                                         (2, 2, 8, "early", "selective"), (2, 3, 4, "on", "selective"),
                                         (4, 2, 4, "off", "selective"), (4, 2, 8, "on", "selective"),
                                         (4, 2, 8, "early", "full"),
                                         (2, 2, 4, "on", "selective-gqa"),  # GQA 4:2 through the exchange
                                         (2, 2, 4, "off", "selective-vp"),  # vocabulary parallelism (§8f)
                                         (4, 2, 8, "off", "full-vp"),
                                         (2, 2, 4, "off", "selective-v2"),  # interleaved v=2 (§8f rank 2)
                                         (2, 1, 4, "off", "full-v2"), (4, 2, 8, "off", "selective-v2"),
                                         (2, 2, 4, "on", "selective-ol"),  # activation offload
                                         (4, 2, 8, "off", "full-ol"),
                                         (4, 2, 8, "early", "selective-xp")])  # exchange placement filter
def test_pipeline_parallel_step_matches_oracle(pp, m, n, x, rc):
    if not torch.cuda.is_available() or torch.cuda.device_count() < pp:
        pytest.skip(f"needs {pp} GPUs")
    gqa, vp, v2, ol = rc.endswith("-gqa"), rc.endswith("-vp"), rc.endswith("-v2"), rc.endswith("-ol")
    xp = rc.endswith("-xp")
    rc = rc.removesuffix("-gqa").removesuffix("-vp").removesuffix("-v2").removesuffix("-ol").removesuffix("-xp")
    env = dict(os.environ, SP_M=str(m), SP_N=str(n), SP_X=x, SP_RC=rc, SP_KV="2" if gqa else "4",
               SP_VP="1" if vp else "0", SP_V="2" if v2 else "1", SP_OFFLOAD="1" if ol else "0",
               SP_XMIN="2" if xp else "0", SP_XSKIP="1" if xp else "0")
    port = 29500 + pp * 100 + m * 10 + n + len(x) + (50 if rc == "full" else 0) + (25 if gqa else 0) + (
        13 if vp else 0) + (37 if v2 else 0) + (61 if ol else 0) + (71 if xp else 0)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={pp}",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        str(ROOT / "tests" / "mp_step_check.py")], env=dict(env, PYTHONUNBUFFERED="1"),
                       capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0
