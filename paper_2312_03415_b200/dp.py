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


def overlapped_backward(run_params: Callable[[], None], run_input: Callable[[], None], g: PackedAdapterGrads,
                        group=None, comm_stream: Optional["torch.cuda.Stream"] = None):
    """Adapter grads -> async allreduce (on `comm_stream` when on CUDA) -> dX.

    Returns the collective's work handle; call .wait() before using g.flat."""
    run_params()
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
