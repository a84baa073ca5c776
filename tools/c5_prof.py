"""Where a C5 stack step's GPU time goes: torch.profiler (CUPTI) kernel totals for the
RunLoRA stack and the default-chain stack (same weights, glue and micro-batches).

    python tools/c5_prof.py [--layers 8] [--micro 2]
Prints one JSON line per arm: total kernel ms per step and the top kernels by time."""
import argparse
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_2312_03415_b200 import runlora as rl  # noqa: E402
from paper_2312_03415_b200.stack import LINEARS, BucketedGradSync, LoRALayer, LoRAStack, plan_model  # noqa: E402
from stack_bench import DefaultLinear, build  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--micro", type=int, default=2)
    ap.add_argument("--no-reuse", action="store_true", help="rebuild W' every micro-batch (no WPrimeCache)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    d, f, r, mb = 4096, 11008, 16, 8192
    model = build(a.layers, d, f, r, dev)
    plan_model(model, mb, rl.BY_TIME)
    model.reuse_wprime_(not a.no_reuse)
    sync = BucketedGradSync.for_model(model)
    g = torch.Generator(device=dev).manual_seed(7)
    xs = [torch.randn(mb, d, generator=g, device=dev).to(torch.bfloat16) for _ in range(a.micro)]
    dys = [torch.randn(mb, d, generator=g, device=dev).to(torch.bfloat16) for _ in range(a.micro)]

    def step_rl():
        sync.begin_step(a.micro)
        for x, dy in zip(xs, dys):
            model(x.detach().requires_grad_(True)).backward(dy)
        sync.finish()

    base = LoRAStack([LoRALayer({nm: DefaultLinear(L.lin[nm]) for nm in LINEARS}) for L in model.layers]).to(dev)

    def step_def():
        for p in base.parameters():
            p.grad = None
        for x, dy in zip(xs, dys):
            base(x.detach().requires_grad_(True)).backward(dy)

    for name, fn in (("runlora", step_rl), ("default", step_def)):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            fn()
        e1.record()
        torch.cuda.synchronize()
        wall = e0.elapsed_time(e1) / 3
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        tot = {}
        for ev in prof.events():
            if ev.device_type == torch.autograd.DeviceType.CUDA:
                key = ev.name[:70]
                t = tot.setdefault(key, [0.0, 0])
                t[0] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
                t[1] += 1
        ksum = sum(v[0] for v in tot.values()) / 1e3
        top = sorted(tot.items(), key=lambda kv: -kv[1][0])[:14]
        print(json.dumps({"arm": name, "reuse_wprime": not a.no_reuse, "layers": a.layers, "micro": a.micro, "ms_per_step_events": wall,
                          "kernel_ms_sum": ksum,
                          "top": [(k, round(v[0] / 1e3, 2), v[1]) for k, v in top]}), flush=True)


if __name__ == "__main__":
    main()
