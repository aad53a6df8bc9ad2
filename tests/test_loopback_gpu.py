"""PP > 1 step parity on ONE GPU: every pipeline rank runs as a host thread
of this process (LoopbackWorld, csrc/host/transport.hpp), so the executor's
multi-stage program — stage sends/receives (reference schedule.cpp:102-130
cross-device edges), the exchange transfers of every tick plan of
apply_exchange (simulator.cpp:56-108: Q/K/V out, attention partials back,
K3 merge, dQ/dK/dV adds), slot arena, recompute — runs on a single-GPU box
exactly as under NCCL, and the assembled model is compared with the float64
oracle (tests/step_parity.py tolerances)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import step_parity as SP
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


def _run(pp, m, n, exchange, recompute, kv_heads=4, interleave=1, **kw):
    from paper_2504_14519_b200.runtime import LoopbackWorld, SlimPipeStep, StepConfig
    cfg = StepConfig.c1(pp=pp, microbatches=m, slices=n, layers=2 * pp * interleave, exchange=exchange,
                        seq_len=1024 * n, recompute=recompute, kv_heads=kv_heads, interleave=interleave, **kw)
    world = LoopbackWorld(pp)
    steps = [SlimPipeStep(cfg, r, pp, loopback=world) for r in range(pp)]
    try:
        tok, tgt = SP.inputs(cfg)
        torch.cuda.synchronize()
        losses = world.run(lambda r: steps[r].step(tok, tgt, optimizer=False), timeout=120, steps=steps)
        assert world.errors() == 0, "loopback transport saw mismatched message sizes"
        allv = [SP.gather_rank(steps[r], cfg, losses[r]) for r in range(pp)]
        ok, worst, _ = SP.compare(cfg, allv, tok, tgt)
        return ok, worst, [s.exchange_stats() for s in steps]
    finally:
        for s in steps:
            s.close()
        world.close()


# (the float64 oracle of an n=8 sequence dominates a case's time, ~40 s)
@pytest.mark.parametrize("pp,m,n,x,rc", [
    (2, 2, 4, "off", "selective"), (2, 1, 2, "off", "full"),
    (2, 2, 4, "on", "full"), (2, 3, 4, "on", "selective"),
    (4, 2, 4, "off", "selective"), (4, 2, 8, "on", "selective"), (4, 2, 8, "early", "full"),
])
def test_loopback_step_matches_oracle(pp, m, n, x, rc):
    _need_gpu()
    ok, worst, xs = _run(pp, m, n, x, rc)
    assert ok, worst
    if x != "off":  # the tick plans really moved attention work
        assert sum(s["passes_out"] for s in xs) > 0 and sum(s["bytes_sent"] for s in xs) > 0


def test_loopback_gqa_through_the_exchange():
    _need_gpu()
    ok, worst, _ = _run(2, 2, 4, "on", "selective", kv_heads=2)
    assert ok, worst


@pytest.mark.parametrize("pp,m,n,rc", [(2, 2, 4, "selective"), (4, 2, 8, "full")])
def test_loopback_interleaved_v2(pp, m, n, rc):
    """Interleaved SlimPipe (v = 2): the stage links form a ring."""
    _need_gpu()
    ok, worst, _ = _run(pp, m, n, "off", rc, interleave=2)
    assert ok, worst


@pytest.mark.parametrize("pp,m,n,rc", [(2, 2, 4, "selective"), (4, 2, 8, "full")])
def test_loopback_vocab_parallel(pp, m, n, rc):
    """Vocabulary parallelism (reference place_vocab distribute=true,
    simulator.cpp:414-522): LM head and cross entropy split over all stages;
    the collectives run as gathers/broadcasts over the loopback links."""
    _need_gpu()
    ok, worst, _ = _run(pp, m, n, "off", rc, vocab=1024, vocab_parallel=True)
    assert ok, worst
