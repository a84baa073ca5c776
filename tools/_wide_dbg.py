import sys, os, torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2312_03415_b200 import runlora as rl
h = rl.handle(0)
cases = [synth.C2[16], synth.C3_UP, synth.C3_DOWN] + [synth.C4[(8, n)] for n in (4096, 32768, 131072)]
for c in cases:
    shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
    X = torch.zeros(c.n, c.k, dtype=torch.bfloat16, device="cuda"); W = torch.zeros(c.k, c.m, dtype=torch.bfloat16, device="cuda")
    A = torch.zeros(c.k, c.r, dtype=torch.bfloat16, device="cuda"); B = torch.zeros(c.r, c.m, dtype=torch.bfloat16, device="cuda")
    dY = torch.zeros(c.n, c.m, dtype=torch.bfloat16, device="cuda")
    Y = torch.empty(c.n, c.m, dtype=torch.bfloat16, device="cuda"); dX = torch.empty(c.n, c.k, dtype=torch.bfloat16, device="cuda")
    dA = torch.empty(c.k, c.r, device="cuda"); dB = torch.empty(c.r, c.m, device="cuda")
    print(c.name, flush=True)
    h.forward(2, shape, X, W, A, B, Y); h.backward(1, shape, X, W, A, B, dY, dX, dA, dB); torch.cuda.synchronize()
