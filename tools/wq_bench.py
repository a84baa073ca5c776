"""Step time with the quantized frozen W (FP8 E4M3 + column scales, R18) vs bf16 W.

    python tools/wq_bench.py [--r 16] [--plan 2,1] [--steps 300]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_03415_b200 import runlora as rl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--r", type=int, default=16)
ap.add_argument("--plan", default="2,1")
ap.add_argument("--steps", type=int, default=300)
a = ap.parse_args()
c = synth.C2[a.r]
d = {k: v.cuda() for k, v in synth.operands(c).items()}
h = rl.handle(0)
shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
ws = h.workspace(shape, True)
Y = torch.empty(c.n, c.m, dtype=torch.bfloat16, device="cuda")
dX = torch.empty(c.n, c.k, dtype=torch.bfloat16, device="cuda")
dA = torch.empty(c.k, c.r, device="cuda")
dB = torch.empty(c.r, c.m, device="cuda")
qw = h.quantize_w(d["W"])
f, b = (int(x) for x in a.plan.split(","))


def bf16_step():
    h.forward(f, shape, d["X"], d["W"], d["A"], d["B"], Y, ws)
    h.backward(b, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, dA, dB, ws=ws)


def wq_step():
    h.forward_wq(f, shape, d["X"], qw, d["A"], d["B"], Y, ws)
    h.backward_wq(b, shape, d["X"], qw, d["A"], d["B"], d["dY"], dX, dA, dB, ws=ws)


def timed(fn):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / a.steps


t_b, t_q, t_b2, t_q2 = timed(bf16_step), timed(wq_step), timed(bf16_step), timed(wq_step)
print(json.dumps({"workload": c.name, "plan": f"F{f}+B{b}", "bf16_W_us": (t_b + t_b2) / 2, "e4m3_W_us": (t_q + t_q2) / 2,
                  "W_bytes_bf16": 2 * c.k * c.m, "W_bytes_e4m3": c.k * c.m + 4 * c.m}))
h.profile_enable(True)
h.profile_read(reset=True)
for _ in range(50):
    wq_step()
torch.cuda.synchronize()
prof = h.profile_read(reset=True)
h.profile_enable(False)
print(json.dumps({k: round(v[1] / v[0] * 1e3, 1) for k, v in prof.items()}))
