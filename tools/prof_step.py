"""Runs forward+backward of one config/plan a few times (driver for ncu captures).

    python tools/prof_step.py --r 16 --plan 1,1 --steps 3 [--config C2|C3_UP|C3_DOWN|C4 --n 32768]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_03415_b200 import runlora as rl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--r", type=int, default=16)
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--plan", default="1,1")
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    c = {"C2": lambda: synth.C2[a.r], "C3_UP": lambda: synth.C3_UP, "C3_DOWN": lambda: synth.C3_DOWN,
         "C4": lambda: synth.C4[(a.r, a.n)]}[a.config]()
    d = {k: v.cuda() for k, v in synth.operands(c).items()}
    h = rl.handle(0)
    shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
    Y = torch.empty(c.n, c.m, dtype=torch.bfloat16, device="cuda")
    dX = torch.empty(c.n, c.k, dtype=torch.bfloat16, device="cuda")
    dA = torch.empty(c.k, c.r, device="cuda")
    dB = torch.empty(c.r, c.m, device="cuda")
    f, b = (int(x) for x in a.plan.split(","))
    for _ in range(a.steps):
        h.forward(f, shape, d["X"], d["W"], d["A"], d["B"], Y)
        h.backward(b, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, dA, dB)
    torch.cuda.synchronize()
    print("ok", c.name, a.plan, h.launch_count())


if __name__ == "__main__":
    main()
