"""Per-launch timeline of forward+backward steps (launch records, RUNLORA_LTRACE=1).

    RUNLORA_LTRACE=1 python tools/step_timeline.py [--plan 2,1] [--r 16] [--steps 20]
For the last --show steps prints, per library launch: first CTA entry, ready (after the
PDL wait: first..last CTA), exit (first..last CTA) relative to the step's first entry,
and the gap between the previous launch's last exit and this launch's first ready.
Numbers in µs.
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_03415_b200 import runlora as rl  # noqa: E402

SIDE = set()  # every library launch is on the caller's stream


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--r", type=int, default=16)
    ap.add_argument("--plan", default="2,1")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--show", type=int, default=2)
    ap.add_argument("--warm", type=int, default=5, help="untimed steps first (1000+: power-capped clocks)")
    ap.add_argument("--shape", default=None, help="n,k,m (default: C2, n=8192, k=m=4096)")
    ap.add_argument("--wq", action="store_true", help="quantized W (FP8 E4M3) entry points")
    a = ap.parse_args()
    assert os.environ.get("RUNLORA_LTRACE"), "set RUNLORA_LTRACE=1"
    c = synth.C2[a.r]
    if a.shape:
        n, k, m = (int(x) for x in a.shape.split(","))
        c = synth.case(f"adhoc_{n}_{k}_{m}_{a.r}", 0, 77, n, k, m, a.r, "bf16")
    d = {k: v.cuda() for k, v in synth.operands(c).items()}
    h = rl.handle(0)
    lib = rl._lib
    lib.runlora_debug_ltrace.restype = C.c_int
    lib.runlora_debug_kernel_name.restype = C.c_char_p
    shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
    ws = h.workspace(shape)
    Y = torch.empty(c.n, c.m, dtype=torch.bfloat16, device="cuda")
    dX = torch.empty(c.n, c.k, dtype=torch.bfloat16, device="cuda")
    dA = torch.empty(c.k, c.r, device="cuda")
    dB = torch.empty(c.r, c.m, device="cuda")
    f, b = (int(x) for x in a.plan.split(","))
    buf = np.zeros(8 * 4096, dtype=np.uint64)
    kids = np.zeros(4096, dtype=np.int32)

    qw = h.quantize_w(d["W"]) if a.wq else None
    if a.wq:
        ws = h.workspace(shape, True)

    def run(k):
        for _ in range(k):
            if qw is not None:
                h.forward_wq(f, shape, d["X"], qw, d["A"], d["B"], Y, ws)
                h.backward_wq(b, shape, d["X"], qw, d["A"], d["B"], d["dY"], dX, dA, dB, ws=ws)
            else:
                h.forward(f, shape, d["X"], d["W"], d["A"], d["B"], Y, ws)
                h.backward(b, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, dA, dB, ws=ws)

    run(a.warm)
    lib.runlora_debug_ltrace(h._h, buf.ctypes.data_as(C.POINTER(C.c_ulonglong)),
                             kids.ctypes.data_as(C.POINTER(C.c_int)), 4096)  # reset
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run(a.steps)
    e1.record()
    torch.cuda.synchronize()
    n = lib.runlora_debug_ltrace(h._h, buf.ctypes.data_as(C.POINTER(C.c_ulonglong)),
                                 kids.ctypes.data_as(C.POINTER(C.c_int)), 4096)
    rec = buf[: 8 * n].reshape(n, 8).astype(np.int64)
    names = [lib.runlora_debug_kernel_name(int(k)).decode() for k in kids[:n]]
    per_step = n // a.steps
    step_us = e0.elapsed_time(e1) * 1e3 / a.steps
    print(f"plan F{f}+B{b}: {per_step} launches/step, {step_us:.1f} us/step (events)")
    # steady-state period from kernel records: first entry of step i -> step i+1
    starts = [rec[i * per_step, 0] for i in range(a.steps)]
    print(f"record period: {np.median(np.diff(starts)) / 1e3:.1f} us/step")
    busy_sum = []
    for s in range(a.steps - a.show, a.steps):
        base = rec[s * per_step, 0]
        last_exit = {"main": None, "side": None}
        print(f"-- step {s}")
        for i in range(s * per_step, (s + 1) * per_step):
            r = rec[i]
            st = "side" if names[i] in SIDE else "main"
            gap = (r[1] - last_exit[st]) / 1e3 if last_exit[st] is not None else float("nan")
            print(f"  {names[i]:16s} {st:4s} entry {(r[0]-base)/1e3:7.1f}  ready {(r[1]-base)/1e3:7.1f}..{(r[2]-base)/1e3:7.1f}"
                  f"  exit {(r[3]-base)/1e3:7.1f}..{(r[4]-base)/1e3:7.1f}  work {(r[4]-r[1])/1e3:6.1f}  gap {gap:5.1f}")
            last_exit[st] = r[4]
    for s in range(a.steps):
        rows = [rec[i] for i in range(s * per_step, (s + 1) * per_step) if names[i] not in SIDE]
        busy_sum.append(sum(r[4] - r[1] for r in rows))
    print(f"main-stream work (ready->last exit) per step: {np.median(busy_sum) / 1e3:.1f} us")


if __name__ == "__main__":
    main()
