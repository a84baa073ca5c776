"""Per-unit timeline of the main GEMM (debug trace, RUNLORA_TRACE=0): for each pair, the
interval between its consecutive tiles' epilogue completions against the tile's load span —
where the exposed epilogue of the 512-wide tiles shows.

    RUNLORA_TRACE=0 python tools/trace_main.py [--M 32768 --N 2048 --K 2048]
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03415_b200 import runlora as rl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=32768)
ap.add_argument("--N", type=int, default=2048)
ap.add_argument("--K", type=int, default=2048)
a = ap.parse_args()
h = rl.handle(0)
f = rl._lib.runlora_debug_gemm
P, I = C.c_void_p, C.c_int
f.restype = I
f.argtypes = [P, I, I, I, P, I, P, I, I, P, P, I, P, P, I, I, I, P]
bf = torch.bfloat16
A = torch.randn(a.M, a.K, device="cuda", dtype=bf)
B = torch.randn(a.N, a.K, device="cuda", dtype=bf)
D = torch.empty(a.M, a.N, device="cuda", dtype=bf)
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    assert f(h._h, a.M, a.N, a.K, A.data_ptr(), 0, B.data_ptr(), 0, 0, A.data_ptr(), B.data_ptr(), 0, D.data_ptr(),
             None, 0, 1, 2, s) == 0, rl._lib.runlora_last_error()
torch.cuda.synchronize()
lib = rl._lib
lib.runlora_debug_trace.restype = C.c_int
buf = np.zeros(8 * 65536 + 4 * 1024, dtype=np.uint64)
n = lib.runlora_debug_trace(h._h, buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), 65536)
t = buf[: 8 * n].reshape(n, 8).astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
T = (t[:, :4] - t0) / 1e3
cta = t[:, 4]
print(f"units {len(t)}  span {T[:, 3].max():.1f} us  CTAs {len(np.unique(cta))}")
loads = T[:, 2] - T[:, 0]
print(f"producer span per unit (start -> last load issued): med {np.median(loads):.2f} us")
gaps, tails = [], []
for c in np.unique(cta):
    s_ = np.sort(np.where(cta == c)[0], kind="stable")
    order = s_[np.argsort(T[s_, 0])]
    done = T[order, 3]
    start = T[order, 0]
    gaps += list(np.diff(done))
    tails += list(done - T[order, 2])
print(f"epilogue done -> next epilogue done on a CTA: med {np.median(gaps):.2f} us  min {np.min(gaps):.2f}  "
      f"max {np.max(gaps):.2f}")
print(f"last load issued -> epilogue done: med {np.median(tails):.2f} us")
last = T[:, 3].max()
firsts = [T[cta == c, 3].max() for c in np.unique(cta)]
print(f"CTA finish spread: {np.min(firsts):.1f} .. {last:.1f} us")
