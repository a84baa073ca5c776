"""Timeline of one traced launch kind (debug trace): RUNLORA_TRACE=<kernel id>, e.g.
2 = rank-r projections, 3 = token reductions (KernelId in csrc/internal.h).

    RUNLORA_TRACE=3 python tools/trace_grads.py [--r 16] [--steps 5]
Prints per-problem unit durations, dependency waits and the number of busy CTAs over time.
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

ap = argparse.ArgumentParser()
ap.add_argument("--r", type=int, default=16)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--plan", default="2,1")
a = ap.parse_args()
c = synth.C2[a.r]
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
lib = rl._lib
lib.runlora_debug_trace.restype = C.c_int
buf = np.zeros(8 * 65536 + 4 * 1024, dtype=np.uint64)
n = lib.runlora_debug_trace(h._h, buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), 65536)
cta = buf[8 * 65536:].reshape(1024, 4).astype(np.int64)
t = buf[: 8 * n].reshape(n, 8).astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
T = (t[:, :4] - t0) / 1e3  # us
print(f"units {len(t)}  span {T[:, 3].max():.1f} us  CTAs {len(np.unique(t[:, 4]))}")
ct = cta[cta[:, 0] > 0]
if len(ct):
    k0 = ct[:, 0].min()
    print(f"kernel: CTA entry {0:.1f}..{(ct[:, 0].max() - k0) / 1e3:.1f} us, inputs ready "
          f"{(ct[:, 1].min() - k0) / 1e3:.1f}..{(ct[:, 1].max() - k0) / 1e3:.1f}, first unit {(t0 - k0) / 1e3:.1f}, "
          f"last unit done {(t[:, 3].max() - k0) / 1e3:.1f}, CTA exit {(ct[:, 2].min() - k0) / 1e3:.1f}.."
          f"{(ct[:, 2].max() - k0) / 1e3:.1f} us")
    # exit time by the number of this launch's CTAs co-resident on the SM
    sm = ct[:, 3]
    cnt = {v: (sm == v).sum() for v in np.unique(sm)}
    per = np.array([cnt[v] for v in sm])
    ex = (ct[:, 2] - ct[:, 1].min()) / 1e3
    for c_ in np.unique(per):
        sel = per == c_
        print(f"  CTAs on an SM = {c_}: {sel.sum():4d} CTAs on {len([v for v in cnt if cnt[v] == c_])} SMs, "
              f"exit after ready med {np.median(ex[sel]):6.1f} min {ex[sel].min():6.1f} max {ex[sel].max():6.1f} us")
    print(f"  SMs used {len(cnt)}")
for q in np.unique(t[:, 5]):
    s = t[:, 5] == q
    wait = T[s, 1] - T[s, 0]
    issue = T[s, 2] - T[s, 1]
    epi = T[s, 3] - T[s, 2]
    print(f"prob {q}: {s.sum():4d} units  start {T[s,0].min():6.1f}..{T[s,0].max():6.1f}  "
          f"dep-wait med {np.median(wait):5.1f} max {wait.max():5.1f}  load-issue med {np.median(issue):5.1f}  "
          f"epi-tail med {np.median(epi):5.1f}  done {T[s,3].min():6.1f}..{T[s,3].max():6.1f}")
# busy CTAs over time (a unit is busy from producer start to epilogue done)
grid = np.arange(0, T[:, 3].max() + 1, 2.0)
for x in grid[::max(1, len(grid) // 25)]:
    busy = ((T[:, 0] <= x) & (T[:, 3] > x)).sum()
    waiting = ((T[:, 0] <= x) & (T[:, 1] > x)).sum()
    print(f"t={x:6.1f} us  active units {busy:4d}  waiting on deps {waiting:4d}")
