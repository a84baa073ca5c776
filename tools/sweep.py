"""Per-config sweep: selected pair (time and FLOP criteria) vs the default XW+(XA)B
autograd chain, on every BASELINE.json bf16 config at 1 GPU.

    python tools/sweep.py [--steps 50] [--only C2] > sweep.jsonl
One JSON line per config: tokens/s and TFLOP/s of the time-selected pair, its plan and
the per-candidate median times, the FLOP pick, the default chain's time, speedup.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_03415_b200 import runlora as rl  # noqa: E402


def timed(fn, steps, warmup=5):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def run(c, steps):
    d = {k: v.cuda() for k, v in synth.operands(c).items()}
    h = rl.handle(0)
    shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
    ws = h.workspace(shape)
    Y = torch.empty(c.n, c.m, dtype=torch.bfloat16, device="cuda")
    dX = torch.empty(c.n, c.k, dtype=torch.bfloat16, device="cuda")
    dA = torch.empty(c.k, c.r, device="cuda")
    dB = torch.empty(c.r, c.m, device="cuda")
    ops = dict(d, Y=Y, dX=dX, dA=dA, dB=dB)
    plan = h.select(shape, rl.BY_TIME, ops=ops, grad_dtype=rl.F32)
    pf = rl.select_by_flops(shape)

    def step(f, b):
        h.forward(f, shape, d["X"], d["W"], d["A"], d["B"], Y, ws)
        h.backward(b, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, dA, dB, ws=ws)

    Xg = d["X"].clone().requires_grad_(True)
    Ag = d["A"].clone().requires_grad_(True)
    Bg = d["B"].clone().requires_grad_(True)

    def default():
        Xg.grad = Ag.grad = Bg.grad = None
        (Xg @ d["W"] + (Xg @ Ag) @ Bg).backward(d["dY"])

    # alternating blocks of the three (clock and power drift hit all alike), medians
    t = {"sel": [], "flops": [], "def": []}
    for _ in range(3):
        t["sel"].append(timed(lambda: step(plan.fwd, plan.bwd), steps))
        t["flops"].append(timed(lambda: step(pf.fwd, pf.bwd), steps))
        t["def"].append(timed(default, steps))
    med = lambda v: sorted(v)[len(v) // 2]  # noqa: E731
    ms, ms_flops, ms_def = med(t["sel"]), med(t["flops"]), med(t["def"])
    fl = plan.flops_fwd[plan.fwd] + plan.flops_bwd[plan.bwd]
    pd = plan.as_dict()
    return {"config": c.name, "n": c.n, "k": c.k, "m": c.m, "r": c.r,
            "plan_time": f"F{plan.fwd}+B{plan.bwd}", "plan_flops": f"F{pf.fwd}+B{pf.bwd}",
            "ms_per_step": ms, "tokens_per_s": c.n / (ms * 1e-3), "tflops": fl / (ms * 1e-3) / 1e12,
            "ms_flops_pick": ms_flops, "ms_default_chain": ms_def, "speedup_vs_default": ms_def / ms,
            "cand_us": {**{f"F{v}": t for v, t in pd["time_fwd_us"].items()},
                        **{f"B{v}": t for v, t in pd["time_bwd_us"].items()}}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--only", default=None)
    ap.add_argument("--per-rank", type=int, default=1,
                    help="divide n by P: one rank's share of a token-sharded run (C4 at P ranks)")
    a = ap.parse_args()
    cfgs = [c for c in synth.ALL_CONFIGS if c.dtype == "bf16"]
    if a.only:
        cfgs = [c for c in cfgs if c.name.startswith(a.only)]
    if a.per_rank > 1:
        cfgs = [synth.case(f"{c.name}_P{a.per_rank}", c.cfg, c.sub, c.n // a.per_rank, c.k, c.m, c.r, c.dtype)
                for c in cfgs]
    for c in cfgs:
        print(json.dumps(run(c, a.steps)), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
