"""forward2 in two halves (include/runlora.h runlora_wprime_t / _wq, runlora_forward_wprime;
Eq. 2) and the W' reuse across micro-batches built on them (lora.WPrimeCache).

1. wprime_t then forward_wprime equals runlora_forward(2) bit for bit (both run the same two
   launches), for bf16 and quantized W, on tile-aligned, ragged and C2 shapes; and the W'ᵀ
   itself equals the fp64 oracle's W + A·B rounded once, within one bf16 rounding.
2. WPrimeCache: a linear used for several micro-batches builds W'ᵀ once, every micro-batch's
   Y equals the uncached forward bit for bit, and an in-place update of A or B (an optimizer
   step) triggers a rebuild whose Y equals a fresh forward with the new adapters.
"""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rl():
    from paper_2312_03415_b200 import runlora
    return runlora


CASES = [synth.case("wp_tiles", 0, 90, 1024, 1024, 512, 16, "bf16"),
         synth.case("wp_ragged", 0, 91, 1000, 1032, 1552, 8, "bf16"),
         synth.C2[16]]


@pytest.mark.parametrize("c", CASES, ids=lambda c: c.name)
def test_two_halves_equal_forward2(rl, c):
    ops = synth.operands(c)
    d = {k: v.cuda() for k, v in ops.items()}
    h = rl.handle(0)
    shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
    ref = torch.empty(c.n, c.m, dtype=torch.bfloat16, device="cuda")
    h.forward(2, shape, d["X"], d["W"], d["A"], d["B"], ref)
    Wpt = torch.full((c.m, c.k), float("nan"), dtype=torch.bfloat16, device="cuda")
    h.wprime_t(shape, d["W"], d["A"], d["B"], Wpt)
    Y = torch.full_like(ref, float("nan"))
    h.forward_wprime(shape, d["X"], Wpt, Y)
    torch.cuda.synchronize()
    assert torch.equal(Y, ref)
    # W'ᵀ against the fp64 definition W + A·B (Eq. 2), one bf16 rounding of the fp32 sum
    W, A, B = (ops[k].double().numpy() for k in ("W", "A", "B"))
    want = (W + A @ B).T
    got = Wpt.double().cpu().numpy()
    assert np.all(np.abs(got - want) <= 2.0 ** -8 * np.abs(want) + 1e-6)
    if c.m % 16 == 0:
        qw = h.quantize_w(d["W"])
        h.forward_wq(2, shape, d["X"], qw, d["A"], d["B"], ref, ws=h.workspace(shape, True))
        h.wprime_t(shape, qw, d["A"], d["B"], Wpt)
        h.forward_wprime(shape, d["X"], Wpt, Y)
        torch.cuda.synchronize()
        assert torch.equal(Y, ref)


def test_two_halves_errors(rl):
    h = rl.handle(0)
    s32 = rl.make_shape(64, 64, 64, 8, rl.F32)
    t = torch.empty(64, 64, device="cuda")
    with pytest.raises(rl.RunLoRAError) as e:
        h.wprime_t(s32, t, t, t, t)
    assert e.value.status == 3  # bf16 only
    s = rl.make_shape(64, 64, 64, 8, rl.BF16)
    with pytest.raises(rl.RunLoRAError) as e:
        rl._check(rl._lib.runlora_wprime_t(h._h, rl.C.byref(s), None, t.data_ptr(), t.data_ptr(), t.data_ptr(),
                                           None), "wprime_t")
    assert e.value.status == 1
    with pytest.raises(rl.RunLoRAError) as e:
        h.forward_wprime(s, t, t, t, ws=torch.empty(16, dtype=torch.uint8, device="cuda"))
    assert e.value.status == 7  # workspace too small


def test_wprime_cache_micro_batches_and_updates(rl):
    from paper_2312_03415_b200.stack import LoRALinear
    c = synth.case("wp_cache", 0, 92, 768, 512, 1024, 16, "bf16")
    ops = synth.operands(c)
    lin = LoRALinear(ops["W"].cuda(), ops["A"].cuda(), ops["B"].cuda(), reuse_wprime=True)
    plain = LoRALinear(ops["W"].cuda(), ops["A"].cuda(), ops["B"].cuda())
    assert plain.wcache is None  # off by default: nothing but W, A, B persists (R20)
    lin.plan = plain.plan = (2, 1)
    X = ops["X"].cuda()
    chunks = [X[i:i + 256] for i in range(0, c.n, 256)]
    for step in range(3):
        for x in chunks:
            y = lin(x.detach().requires_grad_(True))
            y0 = plain(x.detach().requires_grad_(True))
            assert torch.equal(y, y0), step
        assert lin.wcache.builds == step + 1  # once per step, not per micro-batch
        with torch.no_grad():  # the optimizer step: in-place updates bump the version counters
            for m in (lin, plain):
                (m.A if step % 2 == 0 else m.B).add_(0.01)
    torch.cuda.synchronize()
    # a new W (e.g. reloaded) is noticed too
    lin.W = lin.W.clone()
    plain.W = lin.W
    y = lin(chunks[0])
    assert torch.equal(y, plain(chunks[0])) and lin.wcache.builds == 4
    # a quantized W keeps its smaller footprint: no cache
    assert lin.quantize_().wcache is None
