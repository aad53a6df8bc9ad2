"""The executor's enqueue program is deadlock-free under the stream model
(tests/stream_model.py): two-deep link rings, per-direction link streams,
CUDA-event ordering, FIFO NCCL pairing per link, all-rank collectives, and a
bounded host enqueue queue.  Covers v = 1, interleaved v = 2 (ring links),
vocabulary parallelism and the exchange (the executor's own wiring, with and
without the placement filter and just-in-time posting); a negative control
shows the model does detect a cross-rank ordering fault, and it reproduces
the one stall measured on hardware this round."""
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


# ---- the exchange (K4), with the executor's own wiring ----------------------
# The exchange ops come from sp_exchange_passes_json — the per-pass transfer
# lists sp_runtime_create builds (csrc/host/xplan.hpp) — not from a restatement.

@pytest.mark.parametrize("p,m,n,mode", [(2, 2, 4, "on"), (2, 4, 8, "early"), (4, 2, 8, "on"), (4, 4, 8, "early"),
                                        (4, 4, 16, "on"), (8, 2, 16, "early")])
@pytest.mark.parametrize("min_chunks,skip_last", [(0, False), (2, True)])
def test_exchange_program_is_deadlock_free(p, m, n, mode, min_chunks, skip_last):
    for serve_jit in (True, False):  # serves posted at the receiving pass (default) / from the host's run-ahead
        for jit_recv in (True, False):
            assert not SM.exchange_deadlocks(p, m, n, mode, min_chunks, skip_last, serve_jit=serve_jit,
                                             jit_recv=jit_recv)


def test_model_reproduces_the_measured_vocab_parallel_exchange_stall():
    """Vocabulary parallelism with the exchange on stalled at PP=4 on 4 GPUs
    (profiles/r02_parity_logs/multigpu_4gpu_nccl.log: rank 3's device in
    F(1,6,4), ranks 0-2 in VocabForward(1,6)); the model deadlocks in exactly
    that state — rank 0 serves rank 1's request first on its class stream,
    rank 1's request waits behind its compute stream, parked at the vocab
    broadcast, which needs rank 3, which waits for rank 0's partial — and the
    runtime therefore rejects the combination at create (test_abi.py)."""
    st = SM.exchange_deadlocks(4, 2, 8, "on", vp=True)
    assert st
    assert [st[(r, "comp")][3] for r in range(4)] == [(4, 1, 6, 4)] * 3 + [(0, 1, 6, 4)]
    assert all(st[(r, "vocab")][2] == ("bcast", 1, 6) for r in range(4))
    assert not SM.exchange_deadlocks(4, 2, 8, "on")  # the same plan without vocabulary parallelism
