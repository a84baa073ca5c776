"""Host-side cost of the ABI calls (no device sync): µs per forward / backward call.

    python tools/host_overhead.py [--shape 512,2048,2048] [--r 8] [--plan 1,1]
"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_03415_b200 import runlora as rl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="512,2048,2048")
ap.add_argument("--r", type=int, default=8)
ap.add_argument("--plan", default="1,1")
ap.add_argument("--iters", type=int, default=200)
a = ap.parse_args()
n, k, m = (int(x) for x in a.shape.split(","))
c = synth.case("host", 0, 78, n, k, m, a.r, "bf16")
d = {kk: v.cuda() for kk, v in synth.operands(c).items()}
h = rl.handle(0)
shape = rl.make_shape(n, k, m, a.r, rl.BF16)
ws = h.workspace(shape)
Y = torch.empty(n, m, dtype=torch.bfloat16, device="cuda")
dX = torch.empty(n, k, dtype=torch.bfloat16, device="cuda")
dA = torch.empty(k, a.r, device="cuda")
dB = torch.empty(a.r, m, device="cuda")
f, b = (int(x) for x in a.plan.split(","))
for _ in range(10):
    h.forward(f, shape, d["X"], d["W"], d["A"], d["B"], Y, ws)
    h.backward(b, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, dA, dB, ws=ws)
torch.cuda.synchronize()
# enqueue far ahead of the GPU? measure pure host time per call with the GPU idle-ish
tf = tb = 0.0
for _ in range(a.iters):
    t0 = time.perf_counter()
    h.forward(f, shape, d["X"], d["W"], d["A"], d["B"], Y, ws)
    t1 = time.perf_counter()
    h.backward(b, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, dA, dB, ws=ws)
    t2 = time.perf_counter()
    tf += t1 - t0
    tb += t2 - t1
    torch.cuda.synchronize()
print(f"host µs per call: forward {tf / a.iters * 1e6:.1f}, backward {tb / a.iters * 1e6:.1f} "
      f"({h.launch_count()} launches so far)")
