"""Autograd integration: a LoRA linear whose forward/backward run through the
C ABI with the plan chosen by the selector.

Paper: "neither forward function in RunLoRA saves result of XA to context"
— the context holds X (and references to the frozen W and the adapters A, B);
the backward recomputes whatever bracketing it needs (Alg. 1-5).
Layouts follow the paper: X[n,k], W[k,m], A[k,r], B[r,m] (Y = XW).
"""
from __future__ import annotations

import torch

from . import runlora as rl


def _shape(X, W, A):
    n, k = X.shape
    m = W.shape[1]
    r = A.shape[1]
    return rl.make_shape(n, k, m, r, X.dtype)


def _is_q(W):
    return isinstance(W, rl.QuantizedWeight)


class GradSink:
    """fp32 destination of one linear's adapter gradients (views dA [k, r], dB [r, m], e.g.
    into a data-parallel bucket): the backward accumulates into them (micro-batching,
    SURVEY §8(e) "C5") instead of returning A.grad / B.grad, then calls ``on_ready``."""

    def __init__(self, dA: torch.Tensor, dB: torch.Tensor, on_ready=None):
        self.dA, self.dB, self.on_ready = dA, dB, on_ready
        self.accumulate = False  # set True after the first micro-batch of a step

    def ready(self):
        self.accumulate = True
        if self.on_ready is not None:
            self.on_ready(self)


class WPrimeCache:
    """forward2's W'ᵀ = (W + A·B)ᵀ kept between calls while W, A and B are unchanged — the
    micro-batches of one gradient-accumulation step build it once instead of once per
    micro-batch (runlora_wprime_t, then runlora_forward_wprime per call: together forward2
    bit for bit, include/runlora.h).  Validity is keyed on the tensors' storage and torch's
    in-place version counters, so an optimizer step (an in-place update of A or B) or a new
    W rebuilds it; updates through ``.data`` bypass the version counter — call
    ``invalidate()`` after those."""

    def __init__(self):
        self.Wpt = None
        self.key = None
        self.builds = 0

    def invalidate(self):
        self.key = None

    def get(self, h, shape, W, A, B) -> torch.Tensor:
        w = W.q if _is_q(W) else W
        # W' does not depend on the token count n
        key = (w.data_ptr(), w._version, A.data_ptr(), A._version, B.data_ptr(), B._version,
               shape.k, shape.m, shape.r)
        if key != self.key:
            k, m = shape.k, shape.m
            if self.Wpt is None or tuple(self.Wpt.shape) != (m, k) or self.Wpt.device != A.device:
                self.Wpt = torch.empty(m, k, dtype=A.dtype, device=A.device)
            h.wprime_t(shape, W, A, B, self.Wpt)
            self.key = key
            self.builds += 1
        return self.Wpt


class LoRALinearFunction(torch.autograd.Function):
    """Y = LoRA(X) with forward variant plan.fwd and backward variant plan.bwd.
    With a GradSink the adapter gradients go to the sink (fp32) and A.grad/B.grad stay None.
    With a WPrimeCache, forward2 reuses W'ᵀ while W, A and B are unchanged."""

    @staticmethod
    def forward(ctx, X, W, A, B, fwd: int, bwd: int, sink: GradSink | None = None,
                wcache: WPrimeCache | None = None):
        # W: a frozen bf16/fp32 tensor, or an rl.QuantizedWeight (FP8 E4M3 + column scales)
        for t, name in ((X, "X"), (W.q if _is_q(W) else W, "W"), (A, "A"), (B, "B")):
            if not t.is_cuda or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous CUDA tensor")
        shape = _shape(X, W, A)
        h = rl.handle(X.device)
        Y = torch.empty(X.shape[0], W.shape[1], dtype=X.dtype, device=X.device)
        if wcache is not None and fwd == 2 and X.dtype == torch.bfloat16:
            h.forward_wprime(shape, X, wcache.get(h, shape, W, A, B), Y)
        elif _is_q(W):
            h.forward_wq(fwd, shape, X, W, A, B, Y)
        else:
            h.forward(fwd, shape, X, W, A, B, Y)
        if _is_q(W):
            ctx.wq = W
            ctx.save_for_backward(X, A, B)  # no XA; W stays quantized
        else:
            ctx.wq = None
            ctx.save_for_backward(X, W, A, B)   # no XA
        ctx.bwd = bwd
        ctx.sink = sink
        ctx.need_dx = ctx.needs_input_grad[0]
        return Y

    @staticmethod
    def backward(ctx, dY):
        if ctx.wq is not None:
            X, A, B = ctx.saved_tensors
            W = ctx.wq
            run = rl.handle(X.device).backward_wq
        else:
            X, W, A, B = ctx.saved_tensors
            run = rl.handle(X.device).backward
        dY = dY.contiguous()
        shape = _shape(X, W, A)
        dX = torch.empty_like(X) if ctx.need_dx else None
        sink = ctx.sink
        if sink is not None:
            run(ctx.bwd, shape, X, W, A, B, dY, dX, sink.dA, sink.dB, accumulate=sink.accumulate)
            sink.ready()
            return dX, None, None, None, None, None, None, None
        gdt = torch.float32 if X.dtype == torch.float32 else A.dtype
        dA = torch.empty(A.shape, dtype=gdt, device=X.device)
        dB = torch.empty(B.shape, dtype=gdt, device=X.device)
        run(ctx.bwd, shape, X, W, A, B, dY, dX, dA, dB)
        return dX, None, dA.to(A.dtype), dB.to(B.dtype), None, None, None, None


def lora_linear(X, W, A, B, plan=None, criterion=rl.BY_FLOPS):
    """Functional entry: selects the (forward, backward) pair for this shape and applies it.
    BY_FLOPS: Table 1 (host only).  BY_TIME / HYBRID: the library times the candidates once
    per shape on scratch operands of this shape (then serves the cached plan)."""
    if plan is None:
        shape = _shape(X, W, A)
        if criterion == rl.BY_FLOPS:
            plan = rl.select_by_flops(shape)
        else:
            n, k = X.shape
            m, r = W.shape[1], A.shape[1]
            dev, dt = X.device, X.dtype
            Wt = torch.randn(k, m, device=dev, dtype=dt) if _is_q(W) else W  # timing stand-in
            ops = {"X": X.detach(), "W": Wt, "A": A.detach(), "B": B.detach(),
                   "dY": torch.randn(n, m, device=dev, dtype=dt), "Y": torch.empty(n, m, device=dev, dtype=dt),
                   "dX": torch.empty(n, k, device=dev, dtype=dt),
                   "dA": torch.empty(k, r, device=dev), "dB": torch.empty(r, m, device=dev)}
            plan = rl.handle(dev).select(shape, criterion, ops=ops, grad_dtype=rl.F32)
    return LoRALinearFunction.apply(X, W, A, B, int(plan.fwd), int(plan.bwd))
