"""GPU parity of the quantized frozen weight (QLoRA-style; R18)
through the C ABI:

* runlora_quantize_w_e4m3 is bit-exact against the oracle's quantizer (oracle/quant.py,
  written from the E4M3 definition) on the same bf16 W — bytes and scales;
* the W~ the x1 variants multiply by (written by the FP8 identity-tail GEMM, no separate
  dequantization kernel) is bit-exact against the oracle's W~;
* every forward/backward variant through the _wq entry points matches the fp64 oracle of
  Eq. 1-3 evaluated with W~ (relative Frobenius <= 2e-2), small shapes in full and the C2
  shape on sampled rows; the autograd op accepts a QuantizedWeight.
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from oracle import quant as Q

pytestmark = pytest.mark.gpu
TOL = 2e-2


@pytest.fixture(scope="module")
def rl():
    from paper_2312_03415_b200 import runlora
    return runlora


def _np(t):
    return t.detach().to(torch.float64).cpu().numpy()


CASES = [synth.case("q_tiles", 0, 30, 520, 512, 768, 16, "bf16"),
         synth.case("q_ragged_r8", 0, 31, 1000, 1024, 272, 8, "bf16")]


@pytest.mark.parametrize("c", CASES, ids=lambda c: c.name)
def test_quantize_and_dequantize_bit_exact(rl, c):
    ops = synth.operands(c)
    W = ops["W"]
    W[:, 5] = 0  # an all-zero column: scale 1, codes 0
    h = rl.handle(0)
    qw = h.quantize_w(W.cuda())
    torch.cuda.synchronize()
    q_o, s_o = Q.quantize_w(W.double().numpy())
    assert np.array_equal(qw.q.cpu().numpy(), q_o)
    assert np.array_equal(qw.scale.cpu().numpy(), s_o)
    # the scale diagonal, decoded from the E5M2 definition (bias 15, 2 mantissa bits)
    def e5m2(b):
        e, mnt = (b >> 2) & 0x1F, b & 3
        return (mnt / 4) * 2.0 ** -14 if e == 0 else (1 + mnt / 4) * 2.0 ** (e - 15)
    D = qw.diag.cpu().numpy()
    assert D.shape == (c.m, 128)
    for j in range(c.m):
        assert e5m2(int(D[j, j % 128])) == s_o[j], j
        assert np.count_nonzero(D[j]) == 1

    # forward1 multiplies by W~ itself: the converter leaves it after the regular workspace
    shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
    ws = torch.zeros(rl.workspace_size_wq(shape), dtype=torch.uint8, device="cuda")
    d = {k: v.cuda() for k, v in ops.items()}
    Y = torch.empty(c.n, c.m, dtype=torch.bfloat16, device="cuda")
    h.forward_wq(1, shape, d["X"], qw, d["A"], d["B"], Y, ws=ws)
    torch.cuda.synchronize()
    main = rl.workspace_size(shape)
    Wd = ws[main:main + 2 * c.k * c.m].view(torch.bfloat16).view(c.k, c.m)
    assert np.array_equal(_np(Wd), Q.dequantize_w(q_o, s_o))


@pytest.mark.parametrize("c", CASES, ids=lambda c: c.name)
def test_wq_all_variants_match_oracle(rl, c):
    ops = synth.operands(c)
    d = {k: v.cuda() for k, v in ops.items()}
    h = rl.handle(0)
    qw = h.quantize_w(d["W"])
    q_o, s_o = Q.quantize_w(ops["W"].double().numpy())
    Wd = Q.dequantize_w(q_o, s_o)
    X, A, B, dY = (_np(ops[k]) for k in ("X", "A", "B", "dY"))
    shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
    wY = O.forward(1, X, Wd, A, B)
    wA, wB, wX = O.reference_backward(X, Wd, A, B, dY)
    errs = {}
    for f in (1, 2):
        Y = torch.full((c.n, c.m), float("nan"), dtype=torch.bfloat16, device="cuda")
        h.forward_wq(f, shape, d["X"], qw, d["A"], d["B"], Y)
        torch.cuda.synchronize()
        errs[f"F{f}"] = O.rel_fro(_np(Y), wY)
    for b in (1, 2, 3, 4, 5):
        dX = torch.full((c.n, c.k), float("nan"), dtype=torch.bfloat16, device="cuda")
        dA = torch.full((c.k, c.r), float("nan"), device="cuda")
        dB = torch.full((c.r, c.m), float("nan"), device="cuda")
        h.backward_wq(b, shape, d["X"], qw, d["A"], d["B"], d["dY"], dX, dA, dB)
        torch.cuda.synchronize()
        errs[f"B{b}"] = max(O.rel_fro(_np(dA), wA), O.rel_fro(_np(dB), wB), O.rel_fro(_np(dX), wX))
    assert all(e <= TOL for e in errs.values()), errs
    assert max(errs.values()) < 5e-3, errs


def test_wq_c2_sampled_and_autograd(rl):
    from paper_2312_03415_b200.lora import LoRALinearFunction
    c = synth.C2[16]
    ops = synth.operands(c)
    d = {k: v.cuda() for k, v in ops.items()}
    h = rl.handle(0)
    qw = h.quantize_w(d["W"])
    Wd = Q.dequantize_w(qw.q.cpu().numpy(), qw.scale.cpu().numpy())
    rows = synth.sample_rows(c.n, seed_cfg=77)
    X = d["X"].clone().requires_grad_(True)
    A = d["A"].clone().requires_grad_(True)
    B = d["B"].clone().requires_grad_(True)
    Y = LoRALinearFunction.apply(X, qw, A, B, 2, 1)
    Y.backward(d["dY"])
    torch.cuda.synchronize()
    An, Bn = _np(ops["A"]), _np(ops["B"])
    assert O.rel_fro(_np(Y[torch.as_tensor(rows, device="cuda")]), O.forward_rows(_np(ops["X"][rows]), Wd, An, Bn)) <= TOL
    assert O.rel_fro(_np(X.grad[torch.as_tensor(rows, device="cuda")]), O.dX_rows(_np(ops["dY"][rows]), Wd, An, Bn)) <= TOL
    wA, wB = O.adapter_grads(ops["X"].float().numpy(), An, Bn, ops["dY"].float().numpy())
    assert O.rel_fro(_np(A.grad), wA) <= TOL and O.rel_fro(_np(B.grad), wB) <= TOL


def test_wq_errors(rl):
    h = rl.handle(0)
    W = torch.randn(64, 12, device="cuda").to(torch.bfloat16)
    with pytest.raises(rl.RunLoRAError) as e:
        h.quantize_w(W)
    assert e.value.status == 6  # m not a multiple of 16
    c = CASES[0]
    shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
    qw = h.quantize_w(torch.randn(c.k, c.m, device="cuda").to(torch.bfloat16))
    small = torch.empty(rl.workspace_size(shape), dtype=torch.uint8, device="cuda")
    X = torch.randn(c.n, c.k, device="cuda").to(torch.bfloat16)
    A = torch.randn(c.k, c.r, device="cuda").to(torch.bfloat16)
    B = torch.randn(c.r, c.m, device="cuda").to(torch.bfloat16)
    Y = torch.empty(c.n, c.m, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(rl.RunLoRAError) as e:
        h.forward_wq(1, shape, X, qw, A, B, Y, ws=small)
    assert e.value.status == 7
    # the 1-byte Wq needs 16-byte row strides: m a multiple of 16 (bf16 W only needs 8)
    with pytest.raises(rl.RunLoRAError) as e:
        h.quantize_w(torch.randn(256, 264, device="cuda").to(torch.bfloat16))
    assert e.value.status == 6
    s8 = rl.make_shape(64, 256, 264, 8, rl.BF16)
    fake = rl.QuantizedWeight(torch.empty(256, 264, dtype=torch.uint8, device="cuda"),
                              torch.ones(264, device="cuda"), torch.empty(264, 128, dtype=torch.uint8, device="cuda"))
    with pytest.raises(rl.RunLoRAError) as e:
        h.forward_wq(2, s8, X[:64, :256].contiguous(), fake, A[:256, :8].contiguous(), B[:8, :264].contiguous(),
                     torch.empty(64, 264, device="cuda", dtype=torch.bfloat16),
                     ws=torch.empty(rl.workspace_size_wq(s8), dtype=torch.uint8, device="cuda"))
    assert e.value.status == 6
