"""Seeded random shapes through every executable variant vs the fp64 oracle.

The shapes (n, k, m, r; k, m, r multiples of 8 as the bf16 ABI requires) are drawn so
that the plan branches all get visited: rank-r projections with and without K-split bf16
blocks (r in {8, 16, 32} and others), main GEMMs with and without split-K (few tiles at
small n), ragged tails in every dimension, ranks above one MMA tile (r > 256 is left to
test_gpu_parity's r264 case).  Per tensor relative Frobenius error <= 2e-2, healthy < 5e-3.
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth

pytestmark = pytest.mark.gpu

rng = np.random.default_rng(2312)
SHAPES = []
for i in range(14):
    n = int(rng.choice([1, 17, 96, 300, 640, 1000, 2048, 3000]))
    k = int(rng.integers(1, 80)) * 8
    m = int(rng.integers(1, 80)) * 8
    r = int(rng.choice([8, 16, 24, 32, 40, 64, 128]))
    SHAPES.append((i, n, k, m, r))


@pytest.fixture(scope="module")
def rl():
    from paper_2312_03415_b200 import runlora
    return runlora


def _np(t):
    return t.detach().to(torch.float64).cpu().numpy()


@pytest.mark.parametrize("sh", SHAPES, ids=lambda s: "n{}_k{}_m{}_r{}".format(*s[1:]))
def test_fuzz_all_variants(rl, sh):
    i, n, k, m, r = sh
    c = synth.case(f"fuzz{i}", 0, 200 + i, n, k, m, r, "bf16")
    ops = synth.operands(c)
    d = {kk: v.cuda() for kk, v in ops.items()}
    h = rl.handle(0)
    shape = rl.make_shape(n, k, m, r, rl.BF16)
    X, W, A, B, dY = (_np(ops[kk]) for kk in ("X", "W", "A", "B", "dY"))
    wY = O.forward(1, X, W, A, B)
    wA, wB, wX = O.reference_backward(X, W, A, B, dY)
    errs = {}
    for f in (1, 2):
        Y = torch.full((n, m), float("nan"), dtype=torch.bfloat16, device="cuda")
        h.forward(f, shape, d["X"], d["W"], d["A"], d["B"], Y)
        torch.cuda.synchronize()
        errs[f"F{f}"] = O.rel_fro(_np(Y), wY)
    for b in (1, 2, 3, 4, 5):
        dX = torch.full((n, k), float("nan"), dtype=torch.bfloat16, device="cuda")
        dA = torch.full((k, r), float("nan"), device="cuda")
        dB = torch.full((r, m), float("nan"), device="cuda")
        h.backward(b, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, dA, dB)
        torch.cuda.synchronize()
        errs[f"B{b}"] = max(O.rel_fro(_np(dA), wA), O.rel_fro(_np(dB), wB), O.rel_fro(_np(dX), wX))
    bad = {kk: e for kk, e in errs.items() if not e <= 2e-2}
    assert not bad, (sh, errs)
    assert max(errs.values()) < 5e-3, (sh, errs)
