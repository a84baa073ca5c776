"""A forward+backward step of the library captured in a CUDA graph vs the same calls eager.

    python tools/graph_step.py [--shape 512,2048,2048] [--r 8] [--plan 1,1] [--steps 200]
The library's calls are capturable: no host synchronisation inside forward/backward,
kernel arguments (tensor maps included) passed by value, every launch on the caller's
stream; programmatic-dependent-launch edges survive capture.  Checks that the replayed
graph produces the same outputs as the eager calls (bit-exact: same kernels, same order).
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_03415_b200 import runlora as rl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="512,2048,2048")
    ap.add_argument("--r", type=int, default=8)
    ap.add_argument("--plan", default=None, help="fwd,bwd (default: time criterion)")
    ap.add_argument("--steps", type=int, default=200)
    a = ap.parse_args()
    n, k, m = (int(x) for x in a.shape.split(","))
    c = synth.case("graph", 0, 79, n, k, m, a.r, "bf16")
    d = {kk: v.cuda() for kk, v in synth.operands(c).items()}
    h = rl.handle(0)
    shape = rl.make_shape(n, k, m, a.r, rl.BF16)
    ws = h.workspace(shape)
    Y = torch.empty(n, m, dtype=torch.bfloat16, device="cuda")
    dX = torch.empty(n, k, dtype=torch.bfloat16, device="cuda")
    dA = torch.empty(k, a.r, device="cuda")
    dB = torch.empty(a.r, m, device="cuda")
    if a.plan:
        f, b = (int(x) for x in a.plan.split(","))
    else:
        p = h.select(shape, rl.BY_TIME, ops=dict(d, Y=Y, dX=dX, dA=dA, dB=dB), grad_dtype=rl.F32)
        f, b = p.fwd, p.bwd

    def step():
        h.forward(f, shape, d["X"], d["W"], d["A"], d["B"], Y, ws)
        h.backward(b, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, dA, dB, ws=ws)

    def timed(fn, k_):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k_):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / k_

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(5):
            step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    ref = [t.clone() for t in (Y, dX, dA, dB)]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for t in (Y, dX, dA, dB):
        t.zero_()
    g.replay()
    torch.cuda.synchronize()
    same = all(torch.equal(x, y) for x, y in zip(ref, (Y, dX, dA, dB)))
    for _ in range(10):
        g.replay()
        step()
    us_eager = timed(step, a.steps)
    us_graph = timed(g.replay, a.steps)
    print(json.dumps({"shape": [n, k, m, a.r], "plan": f"F{f}+B{b}", "eager_us": us_eager, "graph_us": us_graph,
                      "graph_bit_exact_vs_eager": same}))


if __name__ == "__main__":
    main()
