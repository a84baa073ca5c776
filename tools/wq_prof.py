"""Small driver for profiling the quantized-W builds (ncu -k regex:tc_gemm_kernel): forward2
with bf16 W (W'ᵀ build), forward2 from Wq (fused W'ᵀ), forward1 from Wq (the W~ converter)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_03415_b200 import runlora as rl  # noqa: E402

c = synth.C2[16]
d = {k: v.cuda() for k, v in synth.operands(c).items()}
h = rl.handle(0)
shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
ws = h.workspace(shape, True)
Y = torch.empty(c.n, c.m, dtype=torch.bfloat16, device="cuda")
qw = h.quantize_w(d["W"])
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for _ in range(reps):
    h.forward(2, shape, d["X"], d["W"], d["A"], d["B"], Y, ws)
    h.forward_wq(2, shape, d["X"], qw, d["A"], d["B"], Y, ws)
    h.forward_wq(1, shape, d["X"], qw, d["A"], d["B"], Y, ws)
torch.cuda.synchronize()
print("ok")
