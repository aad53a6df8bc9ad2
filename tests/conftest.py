import os
import sys
from pathlib import Path

# One hardware work queue per CUDA stream (the default 8 makes streams share
# queues, and a waiting stream then stalls unrelated ones; the loopback
# transport runs a dozen streams per rank in one process).  Must be set before
# the CUDA context exists.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session", autouse=True)
def _built_library():
    from paper_2504_14519_b200 import build
    build.build()
    yield
