"""PP > 1 step parity on ONE GPU: every pipeline rank runs as a host thread
of this process (LoopbackWorld, csrc/host/transport.hpp), so the executor's
multi-stage program — stage sends/receives (reference schedule.cpp:102-130
cross-device edges), the exchange transfers of every tick plan of
apply_exchange (simulator.cpp:56-108: Q/K/V out, attention partials back,
K3 merge, dQ/dK/dV adds), slot arena, recompute — runs on a single-GPU box
exactly as under NCCL, and the assembled model is compared with the float64
oracle (tests/step_parity.py tolerances)."""
from __future__ import annotations

import pytest
import torch

from test_attn_gpu import _need_gpu

pytestmark = pytest.mark.gpu


def test_loopback_transport_pingpong_one_thread():
    """Both ranks' operations enqueued by one host thread: the device-side
    protocol alone."""
    _need_gpu()
    from paper_2504_14519_b200.runtime import LoopbackWorld, _lib
    world = LoopbackWorld(2)
    nbytes = 1 << 20
    b = [torch.full((nbytes,), v, dtype=torch.uint8, device="cuda") for v in (1, 2, 0, 0)]
    torch.cuda.synchronize()
    import threading
    rc = [None]
    t = threading.Thread(target=lambda: rc.__setitem__(0, _lib().sp_loopback_pingpong_1thread(
        world.handle, b[0].data_ptr(), b[1].data_ptr(), b[2].data_ptr(), b[3].data_ptr(), nbytes, 4)), daemon=True)
    t.start()
    t.join(60)
    if t.is_alive():
        import os
        import sys
        print("one-thread loopback ping-pong did not finish in 60 s", file=sys.stderr, flush=True)
        os._exit(3)
    assert rc[0] == 0
    assert int(b[2].min()) == 2 and int(b[3].max()) == 1


def test_loopback_transport_pingpong():
    """The transport alone: two threads exchange messages (plain and grouped)
    through device flags and copy kernels; payloads arrive intact."""
    _need_gpu()
    import threading
    from paper_2504_14519_b200.runtime import LoopbackWorld, _lib
    world = LoopbackWorld(2)
    nbytes = 1 << 20
    bufs = [(torch.full((nbytes,), r + 1, dtype=torch.uint8, device="cuda"), torch.zeros(nbytes, dtype=torch.uint8,
                                                                                          device="cuda"))
            for r in range(2)]
    torch.cuda.synchronize()
    rcs = [None, None]

    def body(r):
        rcs[r] = _lib().sp_loopback_pingpong(world.handle, r, bufs[r][0].data_ptr(), bufs[r][1].data_ptr(), nbytes, 8)
    ths = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(2)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(60)
    if any(t.is_alive() for t in ths):
        import os
        import sys
        print("loopback ping-pong did not finish in 60 s", file=sys.stderr, flush=True)
        os._exit(3)
    assert rcs == [0, 0] and world.errors() == 0
    assert int(bufs[0][1].min()) == 2 and int(bufs[1][1].max()) == 1


def _run(pp, m, n, exchange, recompute, kv_heads=4, interleave=1, vocab_parallel=False, env=None):
    """One case in its own process (tests/loopback_step_check.py): a stall
    ends that process and its GPU context, not the session."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    args = [sys.executable, str(root / "tests" / "loopback_step_check.py"), str(pp), str(m), str(n), exchange,
            recompute, str(kv_heads), str(interleave), "1" if vocab_parallel else "0"]
    try:
        r = subprocess.run(args, capture_output=True, text=True, timeout=300,
                           env=dict(os.environ, PYTHONUNBUFFERED="1", **(env or {})))
    except subprocess.TimeoutExpired as e:
        print(e.stdout or "", e.stderr or "")
        return False, "timeout"
    print(r.stdout[-4000:], r.stderr[-3000:])
    worst = [ln for ln in r.stdout.splitlines() if ln.startswith("worst grad err")]
    return r.returncode == 0, worst[-1] if worst else r.returncode


# (the float64 oracle of an n=8 sequence dominates a case's time, ~40 s)
@pytest.mark.parametrize("pp,m,n,x,rc", [
    (2, 2, 4, "off", "selective"), (2, 2, 4, "on", "full"), (2, 2, 8, "early", "selective"),
    (4, 2, 4, "off", "selective"), (4, 2, 8, "on", "selective"),
])
def test_loopback_step_matches_oracle(pp, m, n, x, rc):
    """(the child also checks that exchange on / early really moved work)"""
    _need_gpu()
    ok, worst = _run(pp, m, n, x, rc)
    assert ok, worst


def test_loopback_exchange_placement_filter():
    """The placement filter (slimpipe.h exchange_min_chunks / skip_last):
    only the plan's multi-chunk transfers that avoid the last stage run —
    still parity, still work moved."""
    _need_gpu()
    ok, worst = _run(4, 2, 8, "early", "selective", env={"SP_XMIN": "2", "SP_XSKIP": "1"})
    assert ok, worst


def test_loopback_gqa_through_the_exchange():
    _need_gpu()
    ok, worst = _run(2, 2, 4, "on", "selective", kv_heads=2)
    assert ok, worst


@pytest.mark.parametrize("pp,m,n,rc", [(2, 2, 4, "selective")])
def test_loopback_interleaved_v2(pp, m, n, rc):
    """Interleaved SlimPipe (v = 2): the stage links form a ring."""
    _need_gpu()
    ok, worst = _run(pp, m, n, "off", rc, interleave=2)
    assert ok, worst


@pytest.mark.parametrize("pp,m,n,rc", [(2, 2, 4, "selective")])
def test_loopback_vocab_parallel(pp, m, n, rc):
    """Vocabulary parallelism (reference place_vocab distribute=true,
    simulator.cpp:414-522): LM head and cross entropy split over all stages;
    the collectives run as gathers/broadcasts over the loopback links."""
    _need_gpu()
    ok, worst = _run(pp, m, n, "off", rc, vocab_parallel=True)
    assert ok, worst
