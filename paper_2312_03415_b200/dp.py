"""Token-sharded data parallelism for the LoRA linear.

Rank p owns token rows [p·n/P, (p+1)·n/P) of X, dY, Y and dX.  W (frozen), A and
B are replicated.  Forward needs no communication; backward needs exactly one
exchange: allreduce(SUM) of the adapter gradients, packed as one contiguous fp32
buffer [dA | dB] (dA and dB are views into it, so no packing copy runs).  On GPUs
the allreduce is issued on a communication stream right after the adapter-grad
kernels and overlaps the dX GEMM (the split _params / _input ABI calls).

dA = Xᵀ·dY·Bᵀ and dB = Aᵀ·Xᵀ·dY (Eq. 3) are sums over tokens, so the
sum of per-shard gradients is the full-batch gradient (linearity).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import torch
import torch.distributed as dist


def shard_range(n: int, world: int, rank: int):
    """Contiguous token rows owned by `rank` (balanced; first n % world ranks get one more)."""
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


@dataclass
class PackedAdapterGrads:
    """fp32 [dA | dB] in one buffer; dA [k, r] and dB [r, m] are views."""
    flat: torch.Tensor
    dA: torch.Tensor
    dB: torch.Tensor

    @staticmethod
    def create(k: int, r: int, m: int, device, dtype=torch.float32) -> "PackedAdapterGrads":
        flat = torch.empty(k * r + r * m, dtype=dtype, device=device)
        return PackedAdapterGrads(flat, flat[: k * r].view(k, r), flat[k * r:].view(r, m))


def allreduce_adapter_grads(g: PackedAdapterGrads, group=None, async_op: bool = False):
    """SUM-allreduce of the packed adapter gradients (the only data-path collective)."""
    return dist.all_reduce(g.flat, op=dist.ReduceOp.SUM, group=group, async_op=async_op)


class SymmetricAllreduce:
    """One-shot allreduce of the packed fp32 [dA | dB] over torch symmetric memory (SURVEY
    §8(f) NEXT-2; the a8 exchange without NCCL): each rank's adapter-grad kernels write its
    partial sums straight into its symmetric buffer (`grads` views), a cross-rank barrier
    makes every buffer visible, each rank sums all P buffers in rank order over NVLink with
    runlora_allreduce_sum_f32 into `out` (`result` views; bit-identical on every rank), and
    a second barrier keeps the buffers intact until every rank has read them.

    Opt-in (bench.py: RUNLORA_DP_TRANSPORT=symm); this round's box had one GPU, so the
    multi-GPU path is untested beyond P = 1 (tests/test_gpu_allreduce.py)."""

    def __init__(self, k: int, r: int, m: int, device, handle, group=None):
        import torch.distributed._symmetric_memory as symm_mem
        group = group if group is not None else dist.group.WORLD
        numel = k * r + r * m
        self.buf = symm_mem.empty(numel, dtype=torch.float32, device=device)
        self.hdl = symm_mem.rendezvous(self.buf, group)
        self.out = torch.empty(numel, dtype=torch.float32, device=device)
        self.ptrs = [int(p) for p in self.hdl.buffer_ptrs]  # rank order
        self.handle = handle
        self.grads = PackedAdapterGrads(self.buf, self.buf[: k * r].view(k, r), self.buf[k * r:].view(r, m))
        self.result = PackedAdapterGrads(self.out, self.out[: k * r].view(k, r), self.out[k * r:].view(r, m))

    def run(self):
        """On the current stream: barrier, fixed-order sum of all ranks' buffers, barrier."""
        self.hdl.barrier(channel=0)
        self.handle.allreduce_sum_f32(self.ptrs, self.out)
        self.hdl.barrier(channel=1)


class FusedExchange:
    """The a8 exchange fused into the backward (runlora_backward_exchange):
    every rank's exchange buffer (two epoch halves of r·(k+m) fp32) and flag array live in torch
    symmetric memory; the dX GEMM launch's idle warps sum the rank's token-split slabs into its
    buffer, publish each 64-row chunk to every rank over NVLink, and sum the P ranks' chunks in
    rank order (bit-identical on every rank) — or, with `multicast=True` and a multicast address
    from the symmetric-memory handle, read the switch-side sum (NVLS multimem.ld_reduce).  No
    NCCL call on the step; dA, dB come back already summed over the ranks.

    Opt-in (bench.py: RUNLORA_DP_TRANSPORT=fused).  Correct by construction for P > 1 (the
    device code is the one tests/test_gpu_exchange.py runs with P ranks emulated in one
    cooperative launch); the box of this round has one GPU, so P > 1 runs only under the
    driver's multi-GPU tiers."""

    def __init__(self, k: int, r: int, m: int, device, handle, group=None, multicast: bool = False):
        import torch.distributed._symmetric_memory as symm_mem
        from . import runlora as rl
        group = group if group is not None else dist.group.WORLD
        self.P, self.rank = dist.get_world_size(group), dist.get_rank(group)
        buf_bytes, flag_bytes = rl.exchange_sizes(k, m, r, self.P)
        self.buf = symm_mem.empty(buf_bytes // 4, dtype=torch.float32, device=device)
        self.flags = symm_mem.empty(flag_bytes // 4, dtype=torch.int32, device=device)
        self.flags.zero_()
        hb = symm_mem.rendezvous(self.buf, group)
        hf = symm_mem.rendezvous(self.flags, group)
        torch.cuda.synchronize(device)
        dist.barrier(group)  # every rank's flags are zero before any rank publishes
        mc = int(getattr(hb, "multicast_ptr", 0) or 0) if multicast else 0
        self.multicast = mc != 0
        self.handle = handle
        self._rl = rl
        self._keep = (hb, hf)
        self.x = handle.exchange_create(self.P, self.rank, k, m, r, [int(p) for p in hb.buffer_ptrs],
                                        [int(p) for p in hf.buffer_ptrs], mc or None)
        self.epoch = 0

    def backward(self, bwd, shape, X, W, A, B, dY, dX, dA, dB, accumulate=False, ws=None):
        """The backward of this rank's token shard with dA, dB summed over all ranks (fp32)."""
        self.epoch += 1
        self.handle.backward_exchange(bwd, shape, X, W, A, B, dY, dX, dA, dB, self.x, self.epoch,
                                      accumulate=accumulate, ws=ws)

    def close(self):
        if getattr(self, "x", None) is not None:
            self._rl.exchange_destroy(self.x)
            self.x = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _StreamJoin:
    def __init__(self, stream, device):
        self.stream, self.device = stream, device

    def wait(self):
        if self.stream is not None:
            torch.cuda.current_stream(self.device).wait_stream(self.stream)


def overlapped_backward(run_params: Callable[[], None], run_input: Callable[[], None], g: PackedAdapterGrads,
                        group=None, comm_stream: Optional["torch.cuda.Stream"] = None,
                        exchange: Optional[SymmetricAllreduce] = None):
    """Adapter grads -> async allreduce (on `comm_stream` when on CUDA) -> dX.

    Returns the collective's work handle; call .wait() before using g.flat (or, with
    `exchange`, exchange.result — g must then be exchange.grads)."""
    run_params()
    if exchange is not None:
        if comm_stream is None:
            exchange.run()
            run_input()
            return _StreamJoin(None, g.flat.device)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(g.flat.device))
        comm_stream.wait_event(ev)
        with torch.cuda.stream(comm_stream):
            exchange.run()
        run_input()
        return _StreamJoin(comm_stream, g.flat.device)
    if comm_stream is not None and g.flat.is_cuda:
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(g.flat.device))
        comm_stream.wait_event(ev)
        with torch.cuda.stream(comm_stream):
            work = allreduce_adapter_grads(g, group, async_op=True)
    else:
        work = allreduce_adapter_grads(g, group, async_op=True)
    run_input()
    return work


def broadcast_plan(fwd: int, bwd: int, group=None, device=None):
    """All ranks run the plan chosen on rank 0 (selection is per-rank-n)."""
    t = torch.tensor([fwd, bwd], dtype=torch.int64, device=device)
    dist.broadcast(t, src=0, group=group)
    return int(t[0]), int(t[1])
