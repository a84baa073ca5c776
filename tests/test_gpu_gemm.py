"""Unit tests of the tcgen05 GEMM building block through the runlora_debug_gemm hook.

Each (A major, B major, BN, tail, split, epilogue) combination the variants use is
run on small ragged shapes (several tiles plus a ragged tail in M, N and K) and
compared with an fp64 product of the same bf16 values.
"""
import ctypes as C

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rl():
    from paper_2312_03415_b200 import runlora
    f = runlora._lib.runlora_debug_gemm
    P, I = C.c_void_p, C.c_int
    f.restype = I
    f.argtypes = [P, I, I, I, P, I, P, I, I, P, P, I, P, P, I, I, I, P]
    return runlora


def _run(rl, M, N, K1, a_mn, b_mn, BN, K2=0, out_mode=0, splits=1, seed=0, cg=1):
    g = torch.Generator().manual_seed(seed)
    dev = "cuda"
    bf = torch.bfloat16
    A1 = torch.randn(M, K1, generator=g).to(bf)
    B1 = torch.randn(K1, N, generator=g).to(bf)
    A2 = torch.randn(M, max(K2, 1), generator=g).to(bf)
    B2 = torch.randn(max(K2, 1), N, generator=g).to(bf)
    Cin = torch.randn(M, N, generator=g).to(bf)
    want = A1.double() @ B1.double()
    if K2:
        want = want + A2.double() @ B2.double()
    if out_mode == 1:
        want = want + Cin.double()
    # storage per majorness (see include/runlora_testing.h)
    a_st = (A1.t() if a_mn else A1).contiguous().to(dev)
    b_st = (B1 if b_mn else B1.t()).contiguous().to(dev)
    a2_st = (A2.t() if a_mn else A2).contiguous().to(dev)
    b2_st = (B2 if b_mn else B2.t()).contiguous().to(dev)
    if out_mode == 2:
        nk = (K1 + 63) // 64
        kps = (nk + splits - 1) // splits
        s_eff = (nk + kps - 1) // kps
        D = torch.full((s_eff, M, N), float("nan"), device=dev)
    else:
        D = torch.full((M, N), float("nan"), dtype=bf, device=dev)
    cin = Cin.to(dev)
    h = rl.handle(0)
    st = rl._lib.runlora_debug_gemm(h._h, M, N, K1, a_st.data_ptr(), int(a_mn), b_st.data_ptr(), int(b_mn), K2,
                                    a2_st.data_ptr(), b2_st.data_ptr(), out_mode, D.data_ptr(), cin.data_ptr(), BN,
                                    splits, cg, C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == 0, rl._lib.runlora_last_error()
    torch.cuda.synchronize()
    got = D.double().cpu()
    if out_mode == 2:
        got = got.sum(0)
    err = (got - want).norm() / want.norm()
    return float(err), got, want


CASES = [
    # M, N, K1, a_mn, b_mn, BN, K2
    (128, 256, 64, False, False, 256, 0),
    (128, 256, 64, False, True, 256, 0),
    (128, 128, 64, True, True, 128, 0),
    (300, 520, 200, False, False, 256, 0),
    (300, 520, 200, False, True, 256, 0),
    (296, 200, 264, True, True, 64, 0),
    (328, 64, 1000, True, True, 64, 0),
    (333, 64, 1000, False, True, 64, 0),
    (257, 16, 136, False, False, 16, 0),
    (257, 8, 136, False, False, 16, 0),
    (129, 32, 72, False, False, 32, 0),
    (129, 48, 72, False, False, 48, 0),
    (260, 64, 520, False, False, 64, 0),
    (260, 128, 520, False, False, 128, 0),
    (260, 128, 520, False, True, 128, 0),
    (200, 520, 256, False, True, 256, 16),
    (200, 520, 256, False, False, 256, 16),
    (200, 264, 256, False, False, 256, 128),
    (200, 264, 256, False, True, 256, 72),
    (384, 512, 8, False, True, 256, 0),
    # narrow MN-major B (32B / 64B swizzle)
    (300, 16, 520, False, True, 16, 0),
    (300, 8, 520, False, True, 16, 0),
    (300, 32, 520, False, True, 32, 0),
    (296, 24, 700, True, True, 32, 0),
    (296, 16, 1000, True, True, 16, 0),
]

CASES_CG2 = [
    (256, 256, 64, False, False, 256, 0),
    (256, 256, 64, False, True, 256, 0),
    (520, 776, 328, False, False, 256, 0),
    (520, 776, 328, False, True, 256, 0),
    (300, 520, 256, False, True, 256, 16),
    (300, 520, 256, False, False, 256, 16),
    (300, 264, 256, False, False, 256, 136),
    (512, 512, 1024, True, True, 256, 0),
    (264, 384, 200, True, True, 256, 0),
    (300, 256, 200, False, False, 128, 0),
    (300, 256, 200, False, True, 128, 0),
]


@pytest.mark.parametrize("case", CASES_CG2)
def test_gemm_cta_pair(rl, case):
    M, N, K1, a_mn, b_mn, BN, K2 = case
    err, _, _ = _run(rl, M, N, K1, a_mn, b_mn, BN, K2, cg=2)
    assert err < 8e-3, err


@pytest.mark.parametrize("case", CASES)
def test_gemm_layouts(rl, case):
    M, N, K1, a_mn, b_mn, BN, K2 = case
    err, _, _ = _run(rl, M, N, K1, a_mn, b_mn, BN, K2)
    assert err < 8e-3, err


@pytest.mark.parametrize("splits", [1, 3, 5])
@pytest.mark.parametrize("mn", [(False, True), (True, True), (False, False)])
def test_gemm_splitk_f32(rl, splits, mn):
    a_mn, b_mn = mn
    BN = 64
    err, _, _ = _run(rl, 296, 64 if b_mn else 16, 696, a_mn, b_mn, BN if b_mn else 16, 0, out_mode=2,
                     splits=splits)
    assert err < 1e-5, err


def test_gemm_add_epilogue(rl):
    err, _, _ = _run(rl, 300, 520, 16, False, True, 256, 0, out_mode=1)
    assert err < 8e-3, err
