"""Small-shape driver for compute-sanitizer: every forward/backward variant once on a ragged
bf16 shape and on an fp32 shape (no checking here; the sanitizer reports errors)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_03415_b200 import runlora as rl  # noqa: E402

# ragged bf16; K-split Z blocks + repeated concat tails + in-kernel split fix-up (n = 1024,
# k = m = 512, r = 16: 4 blocks); fp32
for c in (synth.case("san_bf16", 0, 30, 300, 264, 200, 16, "bf16"),
          synth.case("san_zsplit", 0, 32, 1024, 512, 512, 16, "bf16"),
          synth.case("san_f32", 0, 31, 70, 40, 56, 5, "f32")):
    d = {k: v.cuda() for k, v in synth.operands(c).items()}
    h = rl.handle(0)
    shape = rl.make_shape(c.n, c.k, c.m, c.r, c.torch_dtype)
    Y = torch.empty(c.n, c.m, dtype=c.torch_dtype, device="cuda")
    dX = torch.empty(c.n, c.k, dtype=c.torch_dtype, device="cuda")
    dA = torch.empty(c.k, c.r, device="cuda")
    dB = torch.empty(c.r, c.m, device="cuda")
    for f in (1, 2):
        h.forward(f, shape, d["X"], d["W"], d["A"], d["B"], Y)
    for b in range(1, 6):
        h.backward(b, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, dA, dB)
    torch.cuda.synchronize()
    print("ok", c.name, h.launch_count())
