"""C5 stack throughput on one GPU: the RunLoRA stack (paper_2312_03415_b200.stack, plans
chosen per shape) vs the same stack with every linear as the default torch autograd chain
X@W + (X@A)@B.  Same weights, same glue, bf16, n tokens per step.

    python tools/stack_bench.py [--layers 32] [--n 8192] [--r 16] [--steps 5] [--criterion time]
Prints one JSON line.  Weights are drawn on the device with torch's generator (same laws
as synth: Var(W) = Var(A) = 1/k, Var(B) = 1/r) — drawing 12 GB through NumPy would take
minutes; parity of the stack is tests/test_gpu_stack.py's job, this is timing only.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03415_b200 import runlora as rl  # noqa: E402
from paper_2312_03415_b200.stack import LINEARS, LoRALayer, LoRALinear, LoRAStack, plan_model  # noqa: E402


class DefaultLinear(torch.nn.Module):
    def __init__(self, lin: LoRALinear):
        super().__init__()
        self.W, self.A, self.B = lin.W, torch.nn.Parameter(lin.A.detach().clone()), \
            torch.nn.Parameter(lin.B.detach().clone())

    def forward(self, x):
        return x @ self.W + (x @ self.A) @ self.B


def build(layers, d, f, r, dev, seed=2312):
    g = torch.Generator(device=dev).manual_seed(seed)
    dims = {"gate": (d, f), "up": (d, f), "down": (f, d)}
    out = []
    for _ in range(layers):
        lin = {}
        for nm in LINEARS:
            k, m = dims.get(nm, (d, d))
            W = (torch.randn(k, m, generator=g, device=dev) / k ** 0.5).to(torch.bfloat16)
            A = (torch.randn(k, r, generator=g, device=dev) / k ** 0.5).to(torch.bfloat16)
            B = (torch.randn(r, m, generator=g, device=dev) / r ** 0.5).to(torch.bfloat16)
            lin[nm] = LoRALinear(W, A, B)
        out.append(LoRALayer(lin))
    return LoRAStack(out)


def timed(model, x, dy, steps, warmup):
    def step():
        xi = x.detach().requires_grad_(True)
        model(xi).backward(dy)
        for p in model.parameters():
            p.grad = None
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--f", type=int, default=11008)
    ap.add_argument("--r", type=int, default=16)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--criterion", default="time", choices=["flops", "time"])
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    model = build(a.layers, a.d, a.f, a.r, dev)
    plans = plan_model(model, a.n, rl.BY_TIME if a.criterion == "time" else rl.BY_FLOPS)
    g = torch.Generator(device=dev).manual_seed(7)
    x = torch.randn(a.n, a.d, generator=g, device=dev).to(torch.bfloat16)
    dy = torch.randn(a.n, a.d, generator=g, device=dev).to(torch.bfloat16)
    h = rl.handle(dev)
    l0 = h.launch_count()
    ms = timed(model, x, dy, a.steps, a.warmup)
    launches = (h.launch_count() - l0) // (a.steps + a.warmup)
    base = LoRAStack([LoRALayer({nm: DefaultLinear(L.lin[nm]) for nm in LINEARS}) for L in model.layers])
    ms_def = timed(base, x, dy, a.steps, a.warmup)
    flops = 0
    for _, _, lin in model.linears():
        k, m, r = lin.dims
        p = plans[(k, m, r)]
        flops += p.flops_fwd[lin.plan[0]] + p.flops_bwd[lin.plan[1]]
    print(json.dumps({
        "workload": "C5_stack", "layers": a.layers, "n": a.n, "d": a.d, "f": a.f, "r": a.r, "dtype": "bf16",
        "criterion": a.criterion, "plans": {f"{k}x{m}": f"F{int(p.fwd)}+B{int(p.bwd)}" for (k, m, r), p in plans.items()},
        "ms_per_step": ms, "tokens_per_s": a.n / (ms * 1e-3), "tflops": flops / (ms * 1e-3) / 1e12,
        "default_chain_ms": ms_def, "default_chain_tokens_per_s": a.n / (ms_def * 1e-3), "speedup": ms_def / ms,
        "library_launches_per_step": launches,
        "note": "glue (q+k+v, residual adds, gate*up) is torch elementwise in both arms"}), flush=True)


if __name__ == "__main__":
    main()
