"""GPU parity: the CUDA path (through the C ABI) vs the CPU fp64 oracle on the
same seeded inputs.

Tolerances (BASELINE.json north star): relative Frobenius error <= 1e-5 for fp32,
<= 2e-2 for bf16 (fp32 accumulate).  Small shapes are compared in full; the
BASELINE.json configs at full size are compared on sampled rows of Y and dX
(rows the oracle computes one by one) and in full for dA, dB.
"""
import pytest
import torch

import oracle as O
import synth

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-5, "bf16": 2e-2}
FWDS = (1, 2)
BWDS = (1, 2, 3, 4, 5)


@pytest.fixture(scope="module")
def rl():
    from paper_2312_03415_b200 import runlora
    return runlora


def _np(t):
    return t.detach().to(torch.float64).cpu().numpy()


def _dev(ops):
    return {k: v.cuda() for k, v in ops.items()}


def _run_all(rl, c, d, fwds=FWDS, bwds=BWDS, grad_dtype=torch.float32):
    """Runs each variant on device operands d; returns {('F',v): Y, ('B',v): (dA,dB,dX)}."""
    h = rl.handle(0)
    shape = rl.make_shape(c.n, c.k, c.m, c.r, c.torch_dtype)
    out = {}
    for v in fwds:
        Y = torch.full((c.n, c.m), float("nan"), dtype=c.torch_dtype, device="cuda")
        h.forward(v, shape, d["X"], d["W"], d["A"], d["B"], Y)
        out[("F", v)] = Y
    gdt = torch.float32 if c.dtype == "f32" else grad_dtype
    for v in bwds:
        dX = torch.full((c.n, c.k), float("nan"), dtype=c.torch_dtype, device="cuda")
        dA = torch.full((c.k, c.r), float("nan"), dtype=gdt, device="cuda")
        dB = torch.full((c.r, c.m), float("nan"), dtype=gdt, device="cuda")
        h.backward(v, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, dA, dB)
        out[("B", v)] = (dA, dB, dX)
    torch.cuda.synchronize()
    return out


def _check_full(c, ops, out, tol):
    X, W, A, B, dY = (_np(ops[k]) for k in ("X", "W", "A", "B", "dY"))
    errs = {}
    for key, val in out.items():
        if key[0] == "F":
            want = O.forward(key[1], X, W, A, B)
            errs[key] = O.rel_fro(_np(val), want)
        else:
            wA, wB, wX = O.backward(key[1], X, W, A, B, dY)
            gA, gB, gX = (_np(t) for t in val)
            errs[key] = max(O.rel_fro(gA, wA), O.rel_fro(gB, wB), O.rel_fro(gX, wX))
    bad = {k: e for k, e in errs.items() if not (e <= tol)}
    assert not bad, f"{c.name}: {bad} (all: {errs})"
    return errs


# ---------------------------------------------------------------- C1 (fp32)
def test_c1_fp32_all_variants(rl):
    c = synth.C1
    ops = synth.operands(c)
    out = _run_all(rl, c, _dev(ops))
    errs = _check_full(c, ops, out, TOL["f32"])
    assert max(errs.values()) < 2e-6  # healthy-range alarm (true FFMA gives ~3e-7)


# ------------------------------------------------------ small bf16 (full compare)
SMALL = [
    synth.case("ragged_r8", 0, 1, 1000, 1024, 1536, 8, "bf16"),
    synth.case("tiles_r16", 0, 2, 520, 512, 768, 16, "bf16"),
    synth.case("r64", 0, 3, 384, 256, 520, 64, "bf16"),
    synth.case("r128", 0, 4, 300, 384, 256, 128, "bf16"),
    synth.case("r264", 0, 5, 200, 528, 272, 264, "bf16"),
    synth.case("n1", 0, 6, 1, 256, 128, 8, "bf16"),
    synth.case("tiny", 0, 7, 7, 8, 16, 8, "bf16"),
    synth.case("r24_k4096", 0, 8, 640, 4096, 264, 24, "bf16"),
]


@pytest.mark.parametrize("c", SMALL, ids=lambda c: c.name)
def test_small_bf16_all_variants(rl, c):
    ops = synth.operands(c)
    out = _run_all(rl, c, _dev(ops))
    errs = _check_full(c, ops, out, TOL["bf16"])
    assert max(errs.values()) < 5e-3, errs  # healthy-range alarm (SURVEY §8(c) error budget)


def test_small_fp32_ragged(rl):
    c = synth.case("f32_ragged", 0, 9, 333, 200, 150, 5, "f32")
    ops = synth.operands(c)
    _check_full(c, ops, _run_all(rl, c, _dev(ops)), TOL["f32"])


@pytest.mark.parametrize("gdt", [torch.bfloat16, torch.float32])
def test_grad_dtype_and_accumulate(rl, gdt):
    c = SMALL[1]
    ops = synth.operands(c)
    d = _dev(ops)
    h = rl.handle(0)
    shape = rl.make_shape(c.n, c.k, c.m, c.r, c.torch_dtype)
    X, W, A, B, dY = (_np(ops[k]) for k in ("X", "W", "A", "B", "dY"))
    wA, wB, _ = O.reference_backward(X, W, A, B, dY)
    for v in BWDS:
        dA = torch.ones((c.k, c.r), dtype=gdt, device="cuda")
        dB = torch.ones((c.r, c.m), dtype=gdt, device="cuda")
        h.backward(v, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], None, dA, dB, accumulate=True)
        torch.cuda.synchronize()
        assert O.rel_fro(_np(dA), wA + 1.0) <= TOL["bf16"]
        assert O.rel_fro(_np(dB), wB + 1.0) <= TOL["bf16"]


def test_split_backward_matches_full(rl):
    c = SMALL[0]
    ops = synth.operands(c)
    d = _dev(ops)
    h = rl.handle(0)
    shape = rl.make_shape(c.n, c.k, c.m, c.r, c.torch_dtype)
    for v in BWDS:
        full = [torch.empty(s, dtype=dt, device="cuda") for s, dt in
                (((c.k, c.r), torch.float32), ((c.r, c.m), torch.float32), ((c.n, c.k), torch.bfloat16))]
        h.backward(v, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], full[2], full[0], full[1])
        sp = [torch.empty_like(t) for t in full]
        h.backward_params(v, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], sp[0], sp[1])
        h.backward_input(v, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], sp[2])
        torch.cuda.synchronize()
        for a, b in zip(full, sp):
            assert torch.equal(a, b), v


# ------------------------------------------------------------ special cases
@pytest.mark.parametrize("zero", ["A", "B", "X", "dY"])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_special_cases(rl, zero, dtype):
    """exact zeros must come out exactly zero (fp32 accumulation of zeros)."""
    c = synth.case(f"zero_{zero}", 0, 10, 1000, 1024, 1536, 8, dtype) if dtype == "bf16" else \
        synth.case(f"zero_{zero}_f32", 0, 10, 256, 256, 256, 8, "f32")
    ops = synth.operands(c, zero=(zero,))
    out = _run_all(rl, c, _dev(ops))
    _check_full(c, ops, out, TOL[c.dtype])
    for v in BWDS:
        dA, dB, dX = out[("B", v)]
        if zero in ("B", "X", "dY"):
            assert torch.count_nonzero(dA) == 0, (zero, v)
        if zero in ("A", "X", "dY"):
            assert torch.count_nonzero(dB) == 0, (zero, v)
        if zero == "dY":
            assert torch.count_nonzero(dX) == 0
    if zero == "X":
        for v in FWDS:
            assert torch.count_nonzero(out[("F", v)]) == 0


# ------------------------------------------------------------ errors at the ABI
def test_abi_errors(rl):
    h = rl.handle(0)
    c = SMALL[1]
    d = _dev(synth.operands(c))
    shape = rl.make_shape(c.n, c.k, c.m, c.r, c.torch_dtype)
    Y = torch.empty(c.n, c.m, dtype=torch.bfloat16, device="cuda")
    dA = torch.empty(c.k, c.r, device="cuda")
    dB = torch.empty(c.r, c.m, device="cuda")
    dX = torch.empty(c.n, c.k, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(rl.RunLoRAError) as e:
        h.backward(6, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, dA, dB)
    assert e.value.status == 4
    small_ws = torch.empty(1024, dtype=torch.uint8, device="cuda")
    with pytest.raises(rl.RunLoRAError) as e:
        h.forward(1, shape, d["X"], d["W"], d["A"], d["B"], Y, ws=small_ws)
    assert e.value.status == 7
    with pytest.raises(rl.RunLoRAError) as e:
        h.forward(1, rl.make_shape(c.n, c.k + 4, c.m, c.r), d["X"], d["W"], d["A"], d["B"], Y)
    assert e.value.status == 6
    Xoff = torch.empty(c.n * c.k + 8, dtype=torch.bfloat16, device="cuda")[1:1 + c.n * c.k].view(c.n, c.k)
    with pytest.raises(rl.RunLoRAError) as e:
        h.forward(1, shape, Xoff, d["W"], d["A"], d["B"], Y)
    assert e.value.status == 6


# ------------------------------------------------------ BASELINE.json configs
def _sampled_check(rl, c, fwds=FWDS, bwds=BWDS, P=1):
    ops = synth.operands(c)
    d = _dev(ops)
    rows = synth.sample_rows(c.n, P=P, seed_cfg=c.cfg * 100 + c.sub)
    W, A, B = (_np(ops[k]) for k in ("W", "A", "B"))
    Xr = _np(ops["X"][rows])
    dYr = _np(ops["dY"][rows])
    wY = O.forward_rows(Xr, W, A, B)
    wX = O.dX_rows(dYr, W, A, B)
    wA, wB = O.adapter_grads(ops["X"].float().numpy(), A, B, ops["dY"].float().numpy())
    out = _run_all(rl, c, d, fwds, bwds)
    ridx = torch.as_tensor(rows, device="cuda")
    errs = {}
    for key, val in out.items():
        if key[0] == "F":
            errs[key] = O.rel_fro(_np(val[ridx]), wY)
        else:
            gA, gB, gX = val
            errs[key] = max(O.rel_fro(_np(gA), wA), O.rel_fro(_np(gB), wB), O.rel_fro(_np(gX[ridx]), wX))
    bad = {k: e for k, e in errs.items() if not (e <= TOL[c.dtype])}
    assert not bad, f"{c.name}: {bad} (all {errs})"
    assert max(errs.values()) < 5e-3, errs


@pytest.mark.parametrize("c", list(synth.C2.values()) + [synth.C3_UP, synth.C3_DOWN], ids=lambda c: c.name)
def test_baseline_configs_c2_c3(rl, c):
    _sampled_check(rl, c)


@pytest.mark.parametrize("c", list(synth.C4.values()), ids=lambda c: c.name)
def test_baseline_configs_c4(rl, c):
    _sampled_check(rl, c, P=8)


# ------------------------------------------- C4 per-rank shapes under token sharding
# The exact shapes rank p runs at P = 8 (and 2, 4) ranks: n/P rows of C4; at
# these sizes the selector flips to F1+B1 and the main GEMMs take the split-K path.
PER_RANK_FULL = [synth.case(f"C4_rank_n{n}_r{r}", 4, 100 + 3 * j + i, n, 2048, 2048, r, "bf16")
                 for j, n in enumerate((512, 1024, 2048)) for i, r in enumerate((8, 32, 128))]
PER_RANK_SAMPLED = [synth.case(f"C4_rank_n{n}_r{r}", 4, 120 + 3 * j + i, n, 2048, 2048, r, "bf16")
                    for j, n in enumerate((4096, 16384)) for i, r in enumerate((8, 32, 128))]


@pytest.mark.parametrize("c", PER_RANK_FULL, ids=lambda c: c.name)
def test_c4_per_rank_shapes_full(rl, c):
    ops = synth.operands(c)
    errs = _check_full(c, ops, _run_all(rl, c, _dev(ops)), TOL["bf16"])
    assert max(errs.values()) < 5e-3, errs


@pytest.mark.parametrize("c", PER_RANK_SAMPLED, ids=lambda c: c.name)
def test_c4_per_rank_shapes_sampled(rl, c):
    _sampled_check(rl, c)
