"""The executor's enqueue program is deadlock-free under the stream model
(tests/stream_model.py): two-deep link rings, per-direction link streams,
CUDA-event ordering, FIFO NCCL pairing per link, all-rank collectives, and a
bounded host enqueue queue.  Covers v = 1, interleaved v = 2 (ring links) and
vocabulary parallelism; a negative control shows the model does detect a
cross-rank ordering fault."""
import pytest

import stream_model as SM


@pytest.mark.parametrize("p,v,m,n,vp", [(2, 1, 2, 4, False), (2, 1, 4, 8, False), (4, 1, 4, 8, False),
                                        (8, 1, 4, 8, False), (2, 2, 2, 4, False), (4, 2, 2, 8, False),
                                        (2, 1, 2, 4, True), (2, 1, 4, 8, True), (4, 1, 2, 8, True)])
def test_enqueue_program_is_deadlock_free(p, v, m, n, vp):
    assert not SM.deadlocks(p, v, m, n, vp)
    assert not SM.deadlocks(p, v, m, n, vp, host_queue=8)
    assert not SM.deadlocks(p, v, m, n, vp, jit_recv=True)  # the executor's default (SP_JIT_RECV=0: early posts)


def test_model_detects_a_collective_order_fault():
    devs = SM.device_orders(2, 1, 2, 4, True)
    vocab = [x for x, e in enumerate(devs[0]) if e[0] in (4, 5)]
    a, b = vocab[0], vocab[1]  # rank 0 issues its first two vocab collectives swapped
    devs[0][a], devs[0][b] = devs[0][b], devs[0][a]
    ops, _ = SM.build(devs, 2, 1, True)
    assert SM.run(ops, 2)
