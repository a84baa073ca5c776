"""Token-sharded data parallelism on CPU (gloo, world_size 2).

The host-side DP logic of paper_2312_03415_b200.dp (row sharding, packed fp32
[dA | dB] buffer, the single allreduce, overlap ordering, plan broadcast) runs in
two real processes; the oracle stands in for the GPU kernels.  Linearity of
dA = Xᵀ dY Bᵀ and dB = Aᵀ Xᵀ dY over tokens (Eq. 3) means the allreduced
shard gradients must equal the full-batch oracle gradients.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2312_03415_b200 import dp

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, k, m, r, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)  # same full batch on every rank
        X, W, A, B, dY = (rng.standard_normal(s) for s in [(n, k), (k, m), (k, r), (r, m), (n, m)])
        lo, hi = dp.shard_range(n, world, rank)
        f, b = dp.broadcast_plan(*(O.select_by_flops(hi - lo, k, m, r) if rank == 0 else (0, 0)))
        g = dp.PackedAdapterGrads.create(k, r, m, "cpu", dtype=torch.float64)
        out = {}

        def params():
            dA, dB, _ = O.backward(b, X[lo:hi], W, A, B, dY[lo:hi])
            g.dA.copy_(torch.from_numpy(dA))
            g.dB.copy_(torch.from_numpy(dB))

        def inp():
            out["dX"] = O.backward(b, X[lo:hi], W, A, B, dY[lo:hi])[2]
            out["Y"] = O.forward(f, X[lo:hi], W, A, B)

        work = dp.overlapped_backward(params, inp, g)
        work.wait()
        q.put((rank, lo, hi, f, b, g.dA.numpy().copy(), g.dB.numpy().copy(), out["dX"], out["Y"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [64, 37])
def test_dp_allreduce_matches_full_batch(n):
    k, m, r = 24, 40, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(i, WORLD, port, n, k, m, r, q)) for i in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    rng = np.random.default_rng(5)
    X, W, A, B, dY = (rng.standard_normal(s) for s in [(n, k), (k, m), (k, r), (r, m), (n, m)])
    wA, wB, wX = O.reference_backward(X, W, A, B, dY)
    wY = O.forward(1, X, W, A, B)
    plans = {(x[3], x[4]) for x in res}
    assert len(plans) == 1  # every rank runs rank 0's plan
    covered = []
    for rank, lo, hi, f, b, dA, dB, dX, Y in res:
        assert O.rel_fro(dA, wA) <= 1e-12 and O.rel_fro(dB, wB) <= 1e-12
        assert O.rel_fro(dX, wX[lo:hi]) <= 1e-12 and O.rel_fro(Y, wY[lo:hi]) <= 1e-12
        covered.extend(range(lo, hi))
    assert covered == list(range(n))  # shards partition the tokens


def test_shard_range_balanced():
    for n in (1, 7, 8192, 8193):
        for P in (1, 2, 3, 8):
            spans = [dp.shard_range(n, P, p) for p in range(P)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(P - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_packed_grads_are_views():
    g = dp.PackedAdapterGrads.create(3, 2, 5, "cpu")
    g.dA.fill_(1.0)
    g.dB.fill_(2.0)
    assert g.flat[:6].eq(1).all() and g.flat[6:].eq(2).all() and g.flat.numel() == 16


def test_overlapped_backward_exchange_order():
    """With a peer-memory exchange (dp.SymmetricAllreduce, duck-typed here: it needs CUDA),
    overlapped_backward runs adapter grads, then the exchange, then dX, and returns a
    waitable handle (host logic only; the kernel is tests/test_gpu_allreduce.py)."""
    calls = []

    class FakeExchange:
        def run(self):
            calls.append("exchange")

    g = dp.PackedAdapterGrads.create(4, 2, 3, "cpu")
    work = dp.overlapped_backward(lambda: calls.append("params"), lambda: calls.append("input"), g,
                                  exchange=FakeExchange())
    work.wait()
    assert calls == ["params", "exchange", "input"]
