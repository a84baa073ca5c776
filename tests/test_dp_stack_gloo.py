"""C5 data parallelism on CPU (gloo, world_size 2): the bucketed adapter-gradient sync
of paper_2312_03415_b200.stack with two micro-batches per rank.

The oracle stack (oracle/stack.py) stands in for the GPU kernels: every rank computes
its shard's per-linear gradients micro-batch by micro-batch, writes them into the sinks
in backward order with the library's accumulate semantics and marks them ready.  The
buckets' allreduce(SUM) must reproduce the full-batch gradients (linearity over tokens,
Eq. 3), and every bucket's collective must have been launched by the time the
last linear of the last micro-batch is ready.
"""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import stack as S
from paper_2312_03415_b200 import dp
from paper_2312_03415_b200.stack import LINEARS, BucketedGradSync

WORLD = 2
N, D, F, R, NL = 12, 6, 10, 2, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    rng = np.random.default_rng(21)
    dims = {"gate": (D, F), "up": (D, F), "down": (F, D)}
    layers = []
    for _ in range(NL):
        L = {}
        for nm in LINEARS:
            k, m = dims.get(nm, (D, D))
            L[nm] = {"W": rng.standard_normal((k, m)) / np.sqrt(k), "A": rng.standard_normal((k, R)) / np.sqrt(k),
                     "B": rng.standard_normal((R, m)) / np.sqrt(R)}
        layers.append(L)
    return layers, rng.standard_normal((N, D)), rng.standard_normal((N, D))


class _Owner:
    def __init__(self, layer, name):
        self.layer, self.name = layer, name


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        layers, x, dy = _problem()
        order = [(li, nm) for li in range(NL) for nm in LINEARS][::-1]  # backward completion order
        dims = {"gate": (D, F), "up": (D, F), "down": (F, D)}
        items = [((*dims.get(nm, (D, D)), R), _Owner(li, nm)) for li, nm in order]
        sync = BucketedGradSync(items, device="cpu", bucket_bytes=600)  # several buckets
        by_name = {(s.owner.layer, s.owner.name): s for s in sync.sinks}
        lo, hi = dp.shard_range(N, world, rank)
        mid = (lo + hi) // 2
        sync.begin_step(micro_batches=2)
        launched_before_last = None
        for mb, (a, b) in enumerate(((lo, mid), (mid, hi))):
            _, grads = S.stack_backward(dy[a:b], layers, S.stack_forward(x[a:b], layers)[1])
            for i, (li, nm) in enumerate(order):
                s = by_name[(li, nm)]
                gA, gB = (torch.from_numpy(g).float() for g in grads[li][nm])
                if s.accumulate:
                    s.dA.add_(gA)
                    s.dB.add_(gB)
                else:
                    s.dA.copy_(gA)
                    s.dB.copy_(gB)
                if mb == 1 and i == len(order) - 1:
                    launched_before_last = len(sync.works)
                s.ready()
        nb = len(sync.buckets)
        sync.finish()
        out = {(s.owner.layer, s.owner.name): (s.dA.numpy().copy(), s.dB.numpy().copy()) for s in sync.sinks}
        q.put((rank, nb, launched_before_last, out))
    finally:
        dist.destroy_process_group()


def test_bucketed_sync_matches_full_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    layers, x, dy = _problem()
    _, full = S.stack_backward(dy, layers, S.stack_forward(x, layers)[1])
    for rank, nb, launched_before_last, out in res:
        assert nb >= 3
        assert launched_before_last == nb - 1  # all but the last bucket already in flight
        for (li, nm), (gA, gB) in out.items():
            wA, wB = full[li][nm]
            # fp32 buckets: relative Frobenius error at fp32 rounding level
            assert np.linalg.norm(gA - wA) <= 1e-6 * np.linalg.norm(wA), (rank, li, nm)
            assert np.linalg.norm(gB - wB) <= 1e-6 * np.linalg.norm(wB), (rank, li, nm)
