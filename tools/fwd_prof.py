"""Small driver for profiling one forward variant (ncu): RUNLORA_LIB selects the build.

    python tools/fwd_prof.py [--fwd 1] [--reps 4]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_03415_b200 import runlora as rl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--fwd", type=int, default=1)
ap.add_argument("--bwd", type=int, default=0)
ap.add_argument("--reps", type=int, default=4)
a = ap.parse_args()
c = synth.C2[16]
d = {k: v.cuda() for k, v in synth.operands(c).items()}
h = rl.handle(0)
shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
ws = h.workspace(shape)
Y = torch.empty(c.n, c.m, dtype=torch.bfloat16, device="cuda")
dX = torch.empty(c.n, c.k, dtype=torch.bfloat16, device="cuda")
dA = torch.empty(c.k, c.r, device="cuda")
dB = torch.empty(c.r, c.m, device="cuda")
for _ in range(a.reps):
    h.forward(a.fwd, shape, d["X"], d["W"], d["A"], d["B"], Y, ws)
    if a.bwd:
        h.backward(a.bwd, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, dA, dB, ws=ws)
torch.cuda.synchronize()
print("ok", rl.LIB_PATH)
