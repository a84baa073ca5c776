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
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--blocks", type=int, default=20)
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
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / a.steps


# alternating blocks (clock / power drift hits both alike), medians
for fn in (bf16_step, wq_step):
    for _ in range(20):
        fn()
tb, tq = [], []
for _ in range(a.blocks):
    tb.append(timed(bf16_step))
    tq.append(timed(wq_step))
import statistics as st
print(json.dumps({"workload": c.name, "plan": f"F{f}+B{b}", "bf16_W_us": st.median(tb), "e4m3_W_us": st.median(tq),
                  "e4m3_over_bf16": st.median([q / b_ for q, b_ in zip(tq, tb)]), "blocks": a.blocks,
                  "steps_per_block": a.steps, "W_bytes_bf16": 2 * c.k * c.m,
                  "W_bytes_e4m3": c.k * c.m + 4 * c.m + 128 * c.m}))
if os.environ.get("RUNLORA_LTRACE"):  # per-launch in-step work (first ready -> last exit) + gap
    import ctypes as C
    import numpy as np
    lib = rl._lib
    lib.runlora_debug_ltrace.restype = C.c_int
    lib.runlora_debug_kernel_name.restype = C.c_char_p
    buf = np.zeros(8 * 4096, dtype=np.uint64)
    kids = np.zeros(4096, dtype=np.int32)
    args = (h._h, buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), kids.ctypes.data_as(C.POINTER(C.c_int)), 4096)
    for name, fn in (("bf16", bf16_step), ("e4m3", wq_step), ("bf16", bf16_step), ("e4m3", wq_step)):
        lib.runlora_debug_ltrace(*args)
        for _ in range(50):
            fn()
        nrec = lib.runlora_debug_ltrace(*args)
        rec = buf[: 8 * nrec].reshape(nrec, 8).astype(np.int64)
        per = nrec // 50
        rows = []
        for pos in range(per):
            idx = [s_ * per + pos for s_ in range(50)]
            nm = lib.runlora_debug_kernel_name(int(kids[idx[0]])).decode()
            wk = np.median([(rec[j, 4] - rec[j, 1]) / 1e3 for j in idx])
            gp = np.median([(rec[j, 1] - rec[j - 1, 4]) / 1e3 for j in idx if j > 0])
            rows.append(f"{nm}:{wk:.1f}+{gp:.1f}")
        print(name, rows)
