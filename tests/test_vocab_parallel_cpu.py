"""Vocabulary parallelism's host protocol with real collectives, on CPU (gloo,
world size 2 and 4) — SURVEY §8f rank 1.

Each process walks ITS OWN device order of place_vocab(distribute=true) with
the executor's normalised costs (runtime.cpp init) and performs the
VocabForward / VocabBackward collectives in exactly the executor's sequence
(runtime.cpp run_vocab_fwd / run_vocab_bwd): broadcast of the final hidden
state from the last stage, all-reduce MAX of the shard row max, rescale,
all-reduce SUM of (sum of exp, target logit), then the shard's dlogits, a
reduce of the partial dX onto the last stage and the shard's dW.  The float64
numpy arithmetic restates the layers.cu xent_shard_* kernels; the result must
equal the unsharded softmax cross entropy and its gradients (the executor's
non-VP path, layers.cu xent_k).  A mismatch in the collective order across
ranks would hang or mix slices here.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs(m, n, Ls, h, V, seed=0):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((m, n, Ls, h))          # final hidden state per slice (after the final norm)
    W = rng.standard_normal((V, h)) * 0.3           # LM head
    T = rng.integers(0, V, (m, n, Ls))              # targets
    T[:, -1, -1] = -1                               # last token of each microbatch has no target
    return X, W, T


def _worker(rank, world, port, m, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_14519_b200 import plan as P
        Ls, h, V = 8, 6, 20 * world
        Vs, v0 = V // world, rank * (V // world)
        S = Ls * n
        sched = P.place_vocab(world, 1, m, n, True, 1.0 / S, 1.0 / S ** 2, S)
        assert sched["valid"]
        X, W, T = _inputs(m, n, Ls, h, V)
        Wsh = W[v0:v0 + Vs]
        root = world - 1
        stats = {}
        dW = np.zeros_like(Wsh)
        dX = {}
        loss = 0.0
        scale = 1.0 / (m * S)
        for kind, k, i, _stage in sched["order"][rank]:
            if kind == 4:  # VocabForward
                xf = torch.from_numpy(X[k - 1, i - 1].copy() if rank == root else np.zeros((Ls, h)))
                dist.broadcast(xf, root)
                logits = xf.numpy() @ Wsh.T
                m_loc = logits.max(1)
                m_glob = torch.from_numpy(m_loc.copy())
                dist.all_reduce(m_glob, op=dist.ReduceOp.MAX)
                t = T[k - 1, i - 1]
                own = (t >= v0) & (t < v0 + Vs)
                zt = np.stack([np.exp(logits - m_loc[:, None]).sum(1) * np.exp(m_loc - m_glob.numpy()),
                               np.where(own, logits[np.arange(Ls), np.clip(t - v0, 0, Vs - 1)], 0.0)])
                zt = torch.from_numpy(zt)
                dist.all_reduce(zt, op=dist.ReduceOp.SUM)
                stats[(k, i)] = (xf.numpy(), m_glob.numpy(), zt.numpy())
            elif kind == 5:  # VocabBackward
                xf, mg, zt = stats.pop((k, i))
                logits = xf @ Wsh.T
                t = T[k - 1, i - 1]
                prob = np.exp(logits - mg[:, None]) / zt[0][:, None]
                hit = (t[:, None] == np.arange(v0, v0 + Vs)[None, :])
                dlog = (prob - hit) * np.where(t >= 0, scale, 0.0)[:, None]
                if rank == root:
                    loss += float(np.sum(np.where(t >= 0, mg + np.log(zt[0]) - zt[1], 0.0)))
                part = torch.from_numpy(dlog @ Wsh)
                dist.reduce(part, root, op=dist.ReduceOp.SUM)
                if rank == root:
                    dX[(k, i)] = part.numpy()
                dW += dlog.T @ xf
        assert not stats
        allv = [None] * world
        dist.all_gather_object(allv, (dW, dX, loss))
        if rank == 0:
            # unsharded reference (layers.cu xent_k semantics)
            ref_loss, ref_dW = 0.0, np.zeros_like(W)
            worst = 0.0
            for k in range(1, m + 1):
                for i in range(1, n + 1):
                    x, t = X[k - 1, i - 1], T[k - 1, i - 1]
                    lg = x @ W.T
                    mx = lg.max(1)
                    z = np.exp(lg - mx[:, None]).sum(1)
                    p = np.exp(lg - mx[:, None]) / z[:, None]
                    valid = t >= 0
                    ref_loss += float(np.sum(np.where(valid, mx + np.log(z) - lg[np.arange(Ls), np.clip(t, 0, V - 1)],
                                                      0.0)))
                    dl = (p - (t[:, None] == np.arange(V)[None, :])) * np.where(valid, scale, 0.0)[:, None]
                    ref_dW += dl.T @ x
                    worst = max(worst, float(np.abs(allv[-1][1][(k, i)] - dl @ W).max()))
            got_dW = np.concatenate([a[0] for a in allv], 0)
            q.put((abs(allv[-1][2] - ref_loss) / abs(ref_loss), float(np.abs(got_dW - ref_dW).max()), worst,
                   len(allv[-1][1])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m,n", [(2, 2, 4), (2, 3, 8), (4, 2, 8)])
def test_vocab_parallel_protocol_matches_unsharded_cross_entropy(world, m, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
        assert pr.exitcode == 0
    rel_loss, d_w, d_x, slices = q.get(timeout=5)
    assert slices == m * n
    assert rel_loss < 1e-12 and d_w < 1e-12 and d_x < 1e-12
