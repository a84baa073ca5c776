"""C5: a stack of LoRA-adapted linears with Llama-7B projection shapes (BASELINE.json
configs[4]) on top of the C-ABI LoRA linear, with

* model-level planning: one (forward, backward) variant pair per distinct linear shape,
  chosen by the library's selector (FLOP criterion of Table 1, or measured
  time, P:5) — SURVEY §8(f) NEXT-4;
* token-sharded data parallelism whose only exchange is the adapter gradients: every
  linear's fp32 [dA | dB] lives in a bucket; the backward accumulates into it (micro-
  batches) and a bucket's allreduce(SUM) starts as soon as its last linear is done, on a
  communication stream, overlapping the rest of the backward (SURVEY §8(e) "C5").

The per-layer dataflow is DESIGN.md reading R15 (BASELINE.json gives shapes only): Llama's
pre-norm residual block without attention and SiLU, with a weightless RMS normalisation

    h = rms(x);  a = q(h) + k(h) + v(h);  x1 = x + o(a)
    h2 = rms(x1);  x2 = x1 + down(gate(h2) ⊙ up(h2))

The glue (normalisation, sums, the gate product) is plain torch elementwise work around
the hot path; every linear is LoRALinearFunction (Y = XW + (XA)B, Eq. 1, no XA
saved).
"""
from __future__ import annotations

from typing import Dict, List, Optional, Tuple

import torch
import torch.distributed as dist
from torch import nn

from . import runlora as rl
from .lora import GradSink, LoRALinearFunction, WPrimeCache

LINEARS = ("q", "k", "v", "o", "gate", "up", "down")


class LoRALinear(nn.Module):
    """Frozen W [k, m] (paper orientation, Y = XW) with trainable A [k, r], B [r, m].
    ``quantize_()`` replaces W by its FP8 E4M3 form with per-column scales (QLoRA-style,
    DESIGN.md R18); forward and backward then dequantize it per call.
    ``reuse_wprime``: with forward2, W'ᵀ = (W + AB)ᵀ is built once while W, A, B are unchanged
    (the micro-batches of a step; lora.WPrimeCache) — one extra m x k bf16 buffer per linear,
    so off by default (nothing but W, A, B persists between calls, R20) and off for
    a quantized W, whose point is the smaller resident weight."""

    def __init__(self, W: torch.Tensor, A: torch.Tensor, B: torch.Tensor, reuse_wprime: bool = False):
        super().__init__()
        self.register_buffer("W", W)
        self.A = nn.Parameter(A)
        self.B = nn.Parameter(B)
        self.wq: Optional[rl.QuantizedWeight] = None
        self._km = tuple(W.shape)
        self.plan: Tuple[int, int] = (1, 1)
        self.sink: Optional[GradSink] = None
        self.wcache: Optional[WPrimeCache] = WPrimeCache() if reuse_wprime else None

    @property
    def dims(self) -> Tuple[int, int, int]:
        return self._km[0], self._km[1], self.A.shape[1]

    def quantize_(self) -> "LoRALinear":
        self.wq = rl.handle(self.W.device).quantize_w(self.W)
        self.W = None  # only the 8-bit weight and its scales stay resident
        self.wcache = None
        return self

    def forward(self, x):
        fwd, bwd = self.plan
        return LoRALinearFunction.apply(x, self.wq if self.wq is not None else self.W, self.A, self.B, fwd, bwd,
                                        self.sink, self.wcache)


RMS_EPS = 1e-6


def rms(z: torch.Tensor) -> torch.Tensor:
    """Row-wise z / sqrt(mean(z²) + eps) (weightless), fp32 statistics, z's dtype out —
    torch's fused rms_norm (one pass forward and backward) when available."""
    if hasattr(torch.nn.functional, "rms_norm"):
        return torch.nn.functional.rms_norm(z, (z.shape[-1],), None, RMS_EPS)
    zf = z.float()
    return (zf * torch.rsqrt(zf.pow(2).mean(dim=-1, keepdim=True) + RMS_EPS)).to(z.dtype)


class LoRALayer(nn.Module):
    def __init__(self, lin: Dict[str, nn.Module]):
        super().__init__()
        self.lin = nn.ModuleDict(lin)

    def forward(self, x):
        L = self.lin
        h = rms(x)
        a = L["q"](h) + L["k"](h) + L["v"](h)
        x1 = x + L["o"](a)
        h2 = rms(x1)
        return x1 + L["down"](L["gate"](h2) * L["up"](h2))


class LoRAStack(nn.Module):
    def __init__(self, layers: List[LoRALayer]):
        super().__init__()
        self.layers = nn.ModuleList(layers)

    @staticmethod
    def from_weights(weights: List[dict], device) -> "LoRAStack":
        """weights: [{name: {"W", "A", "B"}}] per layer (e.g. synth.c5_weights)."""
        return LoRAStack([LoRALayer({nm: LoRALinear(*(w[nm][t].to(device) for t in ("W", "A", "B")))
                                     for nm in LINEARS}) for w in weights])

    def linears(self) -> List[Tuple[int, str, LoRALinear]]:
        """(layer, name, module) in forward order."""
        return [(i, nm, L.lin[nm]) for i, L in enumerate(self.layers) for nm in LINEARS]

    def reuse_wprime_(self, enable: bool = True) -> "LoRAStack":
        """forward2's W'ᵀ built once per optimizer step per linear and reused by the step's
        micro-batches (one extra m x k bf16 buffer per linear; no effect on quantized linears)."""
        for _, _, lin in self.linears():
            lin.wcache = WPrimeCache() if enable and lin.wq is None else None
        return self

    def quantize_(self) -> "LoRAStack":
        """Every frozen W to FP8 E4M3 + per-column scales (QLoRA-style fine-tuning)."""
        for _, _, lin in self.linears():
            lin.quantize_()
        return self

    def forward(self, x):
        for L in self.layers:
            x = L(x)
        return x


def plan_model(model: LoRAStack, n: int, criterion=rl.BY_FLOPS) -> Dict[Tuple[int, int, int], rl.Plan]:
    """Selects one variant pair per distinct (k, m, r) of the model's linears at n tokens
    and assigns it to every linear of that shape.  BY_TIME / HYBRID time the candidates on
    scratch operands of that shape (the library caches the plan per shape)."""
    plans = {}
    for _, _, lin in model.linears():
        k, m, r = lin.dims
        key = (k, m, r)
        if key not in plans:
            shape = rl.make_shape(n, k, m, r, lin.A.dtype)
            if criterion == rl.BY_FLOPS:
                plans[key] = rl.select_by_flops(shape)
            else:
                dev, dt = lin.A.device, lin.A.dtype
                W = lin.W if lin.W is not None else torch.randn(k, m, device=dev, dtype=dt)  # timing stand-in
                ops = {"X": torch.randn(n, k, device=dev, dtype=dt), "W": W, "A": lin.A.detach(),
                       "B": lin.B.detach(), "dY": torch.randn(n, m, device=dev, dtype=dt),
                       "Y": torch.empty(n, m, device=dev, dtype=dt), "dX": torch.empty(n, k, device=dev, dtype=dt),
                       "dA": torch.empty(k, r, device=dev), "dB": torch.empty(r, m, device=dev)}
                plans[key] = rl.handle(dev).select(shape, criterion, ops=ops, grad_dtype=rl.F32)
        lin.plan = (int(plans[key].fwd), int(plans[key].bwd))
    return plans


class BucketedGradSync:
    """fp32 adapter gradients of every linear, packed into buckets in backward-completion
    order (reverse forward order).  Each linear's GradSink views its slice of a bucket.

    Use per step: ``begin_step(micro_batches)``; run the micro-batches' forward/backward;
    ``finish()`` (waits for the collectives).  The backward of the LAST micro-batch marks
    linears ready; a bucket whose linears are all ready is allreduced right away (async, on
    ``comm_stream`` after an event on the compute stream), overlapping the remaining
    backward.  With world size 1 (or no process group) no collective runs."""

    def __init__(self, sinks_in_order: List[Tuple[Tuple[int, int, int], object]], device, bucket_bytes=25 << 20,
                 group=None, comm_stream=None, always_reduce=False):
        self.device = torch.device(device)
        self.group = group
        self.comm_stream = comm_stream
        self.always_reduce = always_reduce  # run the collectives even in a 1-rank group (tests)
        self.buckets: List[torch.Tensor] = []
        self.members: List[List[GradSink]] = []
        self.sinks: List[GradSink] = []
        self.bucket_of: Dict[int, int] = {}
        cur, cur_elems = [], 0
        groups = []
        for (k, m, r), owner in sinks_in_order:
            e = k * r + r * m
            if cur and (cur_elems + e) * 4 > bucket_bytes:
                groups.append((cur, cur_elems))
                cur, cur_elems = [], 0
            cur.append(((k, m, r), owner))
            cur_elems += e
        if cur:
            groups.append((cur, cur_elems))
        for bi, (items, elems) in enumerate(groups):
            flat = torch.zeros(elems, dtype=torch.float32, device=self.device)
            off, mem = 0, []
            for (k, m, r), owner in items:
                dA = flat[off:off + k * r].view(k, r)
                off += k * r
                dB = flat[off:off + r * m].view(r, m)
                off += r * m
                s = GradSink(dA, dB, on_ready=self._ready)
                s.owner = owner
                self.bucket_of[id(s)] = bi
                mem.append(s)
                self.sinks.append(s)
            self.buckets.append(flat)
            self.members.append(mem)
        self._left: List[int] = []
        self._mb_left = 0
        self.works = []

    @staticmethod
    def for_model(model: LoRAStack, **kw) -> "BucketedGradSync":
        """Attaches a sink to every linear of the model (backward order)."""
        lins = list(reversed(model.linears()))
        sync = BucketedGradSync([(lin.dims, lin) for _, _, lin in lins], device=lins[0][2].A.device, **kw)
        for s in sync.sinks:
            s.owner.sink = s
        return sync

    def _world(self) -> int:
        return dist.get_world_size(self.group) if dist.is_available() and dist.is_initialized() else 1

    def begin_step(self, micro_batches: int = 1):
        for s in self.sinks:
            s.accumulate = False  # the first micro-batch overwrites
        self._left = [len(m) for m in self.members]
        self._mb_left = micro_batches
        self._done_in_mb = 0
        self.works = []

    def _ready(self, sink: GradSink):
        self._done_in_mb += 1
        last_mb = self._mb_left == 1
        if self._done_in_mb == len(self.sinks):  # a micro-batch's backward is complete
            self._done_in_mb = 0
            self._mb_left -= 1
        if not last_mb:
            return
        bi = self.bucket_of[id(sink)]
        self._left[bi] -= 1
        if self._left[bi] == 0 and (self._world() > 1 or (self.always_reduce and dist.is_initialized())):
            self._launch(bi)

    def _launch(self, bi: int):
        flat = self.buckets[bi]
        if self.comm_stream is not None and flat.is_cuda:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(flat.device))
            self.comm_stream.wait_event(ev)
            with torch.cuda.stream(self.comm_stream):
                self.works.append(dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=self.group, async_op=True))
        else:
            self.works.append(dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=self.group, async_op=True))

    def finish(self):
        for w in self.works:
            w.wait()
        if self.comm_stream is not None and self.device.type == "cuda":
            torch.cuda.current_stream(self.device).wait_stream(self.comm_stream)
        self.works = []
