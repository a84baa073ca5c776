"""Long-run determinism at C2 (BASELINE.json configs[1], r = 16): thousands of back-to-back
forward+backward steps through the C ABI must give bit-identical Y, dX, dA and dB on every
step.  Every reduction in the path has a fixed order (TMEM accumulation over a fixed K
sequence, the in-kernel split fix-up summing slabs in split order), so any deviation is a
race — e.g. a shared-memory region reused before an asynchronous reader is done, which in
round 1 surfaced only after ~1000 steps (profiles/r01/SUMMARY.md finding 10)."""
import pytest
import torch

import oracle as O
import synth

pytestmark = pytest.mark.gpu
STEPS = 2000


@pytest.fixture(scope="module")
def rl():
    from paper_2312_03415_b200 import runlora
    return runlora


@pytest.mark.parametrize("plan", [(2, 1), (1, 1), (2, 5)], ids=lambda p: f"F{p[0]}+B{p[1]}")
def test_back_to_back_steps_bit_identical(rl, plan):
    fwd, bwd = plan
    c = synth.C2[16]
    ops = synth.operands(c)
    d = {k: v.cuda() for k, v in ops.items()}
    h = rl.handle(0)
    shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
    ws = h.workspace(shape)
    out = {"Y": torch.empty(c.n, c.m, dtype=torch.bfloat16, device="cuda"),
           "dX": torch.empty(c.n, c.k, dtype=torch.bfloat16, device="cuda"),
           "dA": torch.empty(c.k, c.r, device="cuda"), "dB": torch.empty(c.r, c.m, device="cuda")}

    def step():
        h.forward(fwd, shape, d["X"], d["W"], d["A"], d["B"], out["Y"], ws)
        h.backward(bwd, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], out["dX"], out["dA"], out["dB"], ws=ws)

    step()
    ref = {k: v.clone() for k, v in out.items()}
    bad = torch.zeros((), dtype=torch.int64, device="cuda")
    first_bad = torch.full((), -1, dtype=torch.int64, device="cuda")
    for i in range(STEPS):
        step()
        diff = torch.stack([(out[k] != ref[k]).any() for k in ("Y", "dX", "dA", "dB")]).any()
        first_bad = torch.where(diff & (first_bad < 0), torch.tensor(i, device="cuda"), first_bad)
        bad += diff.long()
    torch.cuda.synchronize()
    assert int(bad) == 0, f"{int(bad)} of {STEPS} steps differed (first at step {int(first_bad)})"
    # and the repeated result is the right one (full dA, dB vs the fp64 oracle)
    W, A, B = (ops[k].double().numpy() for k in ("W", "A", "B"))
    wA, wB = O.adapter_grads(ops["X"].float().numpy(), A, B, ops["dY"].float().numpy())
    assert O.rel_fro(ref["dA"].double().cpu().numpy(), wA) < 5e-3
    assert O.rel_fro(ref["dB"].double().cpu().numpy(), wB) < 5e-3


def test_quantized_w_back_to_back_bit_identical(rl):
    """The quantized-W path (FP8 tail GEMMs building W' / W'ᵀ from Wq, R18) under
    the same long-run determinism check, F2+B5 (its time pick) and F2+B1 (W~ materialised)."""
    c = synth.C2[16]
    d = {k: v.cuda() for k, v in synth.operands(c).items()}
    h = rl.handle(0)
    shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
    qw = h.quantize_w(d["W"])
    ws = h.workspace(shape, quantized_w=True)
    out = {"Y": torch.empty(c.n, c.m, dtype=torch.bfloat16, device="cuda"),
           "dX": torch.empty(c.n, c.k, dtype=torch.bfloat16, device="cuda"),
           "dA": torch.empty(c.k, c.r, device="cuda"), "dB": torch.empty(c.r, c.m, device="cuda")}
    for fwd, bwd in ((2, 5), (2, 1)):
        def step():
            h.forward_wq(fwd, shape, d["X"], qw, d["A"], d["B"], out["Y"], ws=ws)
            h.backward_wq(bwd, shape, d["X"], qw, d["A"], d["B"], d["dY"], out["dX"], out["dA"], out["dB"], ws=ws)

        step()
        ref = {k: v.clone() for k, v in out.items()}
        bad = torch.zeros((), dtype=torch.int64, device="cuda")
        for _ in range(STEPS // 2):
            step()
            bad += torch.stack([(out[k] != ref[k]).any() for k in ("Y", "dX", "dA", "dB")]).any().long()
        torch.cuda.synchronize()
        assert int(bad) == 0, (fwd, bwd, int(bad))
