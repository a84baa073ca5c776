"""Pins for the CPU fp64 oracle (-m "not gpu").

Each test ties the oracle to something other than itself: values printed in the
paper or derived by hand from its equations (tests/golden/), Table 1 evaluated by
SPEC's author, finite differences, the mathematics of Eq. 4 (associativity),
torch autograd of Eq. 1 (an independent library routine), special cases with
closed forms, and the paper's dominance proofs.
"""
import json
import os
import random

import numpy as np
import pytest
import torch

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _rand(rng, *shape):
    return rng.standard_normal(shape)


# ------------------------------------------------------------ worked examples
def test_integer_example_all_variants():
    """tests/golden/integer_example.json: hand-expanded Eq. 1-3 on integers."""
    g = _load("integer_example.json")
    X, W, A, B, dY = (np.array(g[k], dtype=np.float64) for k in ("X", "W", "A", "B", "dY"))
    for v in O.FWD_VARIANTS:
        np.testing.assert_array_equal(O.forward(v, X, W, A, B), np.array(g["Y"]))
    for v in O.BWD_VARIANTS:
        dA, dB, dX = O.backward(v, X, W, A, B, dY)
        np.testing.assert_array_equal(dA, np.array(g["dA"]), err_msg=f"B{v}")
        np.testing.assert_array_equal(dB, np.array(g["dB"]), err_msg=f"B{v}")
        np.testing.assert_array_equal(dX, np.array(g["dX"]), err_msg=f"B{v}")
    np.testing.assert_array_equal(O.forward_rows(X[[2, 0]], W, A, B), np.array(g["Y"])[[2, 0]])
    np.testing.assert_array_equal(O.dX_rows(dY[[1]], W, A, B), np.array(g["dX"])[[1]])
    dA, dB = O.adapter_grads(X, A, B, dY, row_chunk=2)
    np.testing.assert_array_equal(dA, np.array(g["dA"]))
    np.testing.assert_array_equal(dB, np.array(g["dB"]))


def test_scalar_example():
    """S:237 scalar evaluation of Eq. 3."""
    g = _load("scalar_example.json")
    X, W, A, B, dY = (np.array([[float(g[k])]]) for k in ("X", "W", "A", "B", "dY"))
    for v in O.FWD_VARIANTS:
        assert O.forward(v, X, W, A, B)[0, 0] == g["Y"]
    for v in O.BWD_VARIANTS:
        dA, dB, dX = O.backward(v, X, W, A, B, dY)
        assert (dA[0, 0], dB[0, 0], dX[0, 0]) == (g["dA"], g["dB"], g["dX"])


# ------------------------------------------------------------------ Table 1
def test_table1_spec_values():
    g = _load("table1_flops.json")
    for c in g["cases"]:
        n = c["b"] * c["s"]
        k, m, r = c["i"], c["o"], c["r"]
        for key, val in c.items():
            if key.startswith("F") and key[1:].isdigit():
                assert O.flops_forward(int(key[1:]), n, k, m, r) == val, key
            if key.startswith("B") and key[1:].isdigit():
                assert O.flops_backward(int(key[1:]), n, k, m, r) == val, key
        if "baseline_backward" in c:
            assert O.baseline_flops(n, k, m, r)[1] == c["baseline_backward"]
    for s in g["select"]:
        n = s["b"] * s["s"]
        f, b = O.select_by_flops(n, s["i"], s["o"], s["r"])
        assert f == s["fwd"]
        if "bwd" in s:
            assert b == s["bwd"]


AUDIT_SHAPES = [(256, 256, 256, 8), (200, 512, 512, 32), (7, 5, 11, 3), (1, 1, 1, 1),
                (33, 17, 9, 4), (64, 48, 80, 16)]


@pytest.mark.parametrize("shape", AUDIT_SHAPES)
def test_flop_audit(shape):
    """The counting matmul, run through each variant as written in the paper, must
    equal the Table 1 polynomial exactly.  B6: the printed row is
    2·i·o·r larger than its own bracketing (reading R4)."""
    n, k, m, r = shape
    rng = np.random.default_rng(1)
    X, W, A, B, dY = (_rand(rng, *s) for s in [(n, k), (k, m), (k, r), (r, m), (n, m)])
    for v in O.FWD_VARIANTS:
        c = O.Counter()
        O.forward(v, X, W, A, B, c)
        assert c.flops == O.flops_forward(v, n, k, m, r), f"F{v}"
    for v in O.BWD_VARIANTS:
        c = O.Counter()
        O.backward(v, X, W, A, B, dY, c)
        want = O.flops_backward(v, n, k, m, r)
        if v == 6:
            want -= 2 * k * m * r
        assert c.flops == want, f"B{v}"


def test_table1_symbolic_differences():
    """Closed-form differences used in the proofs and crossovers."""
    rng = random.Random(5)
    for _ in range(2000):
        n, k, m, r = (rng.randint(1, 5000) for _ in range(4))
        fb = lambda v: O.flops_backward(v, n, k, m, r)
        ff = lambda v: O.flops_forward(v, n, k, m, r)
        assert ff(2) - ff(1) == -2 * r * (n * (k + m) - k * m)
        assert fb(5) - fb(1) == 2 * k * r * (m - n)
        assert fb(2) - fb(5) == 2 * n * m * (k - r)
        assert fb(3) - fb(5) == 2 * (n * (k * m - k * r - m * r) + k * m * r)
        assert fb(4) - fb(5) == 2 * (n * (k * m - 2 * r * (k + m)) + 2 * k * m * r)
        assert fb(7) == fb(8) == fb(3)
        assert fb(6) > fb(5)


def test_dominance_proofs():
    """under Eq. 5, B2 > B5 and B3 > B5; B6 > B5 always."""
    rng = np.random.default_rng(7)
    N = 100_000
    n = rng.integers(1, 1 << 17, N)
    k = rng.integers(1, 1 << 14, N)
    m = rng.integers(1, 1 << 14, N)
    r = rng.integers(1, 1 << 10, N)
    n, k, m, r = (a.astype(object) for a in (n, k, m, r))
    red = r * (k + m) < k * m
    assert red.sum() > N // 2
    b2 = 2 * n * (m * r + 2 * k * r + 2 * k * m) + 2 * k * m * r
    b3 = 2 * n * (2 * k * m + m * r + k * r) + 4 * k * r * m
    b5 = 2 * n * (2 * m * r + 2 * k * r + m * k) + 2 * k * m * r
    b6 = 2 * n * (2 * m * r + 2 * k * r + 2 * m * k) + 4 * k * m * r
    assert all((b2 > b5)[red]) and all((b3 > b5)[red])
    assert all(b6 > b5)
    # and the oracle's own table agrees on a subsample
    for j in range(0, N, 997):
        assert O.flops_backward(2, n[j], k[j], m[j], r[j]) == b2[j]
        assert O.flops_backward(5, n[j], k[j], m[j], r[j]) == b5[j]


def test_selector_crossovers_fig3():
    """Fig. 3: LlamaMLP 4096->11008, r=128: F1 below n = io/(i+o) ≈ 2985.2,
    F2 above; B1 below n = o = 11008, B5 above (B5-B1 = 2ir(o-n))."""
    k, m, r = 4096, 11008, 128
    assert O.param_reduction(k, m, r)
    assert O.select_by_flops(2985, k, m, r)[0] == 1
    assert O.select_by_flops(2986, k, m, r)[0] == 2
    assert O.select_by_flops(11007, k, m, r)[1] == 1
    assert O.select_by_flops(11008, k, m, r)[1] == 1   # exact tie -> lowest index
    assert O.select_by_flops(11009, k, m, r)[1] == 5
    for n in (1, 10, 600, 2048, 20480, 1 << 20):
        assert O.select_by_flops(n, k, m, r)[1] in (1, 4, 5)


def test_param_reduction():
    assert O.param_reduction(4096, 4096, 128)
    assert not O.param_reduction(2, 2, 1)         # S:140 boundary equality
    assert O.param_reduction(4096, 11008, 128)


def test_workspace_elements():
    assert O.workspace_elements(True, 1, 1, 1, 1, 1) == 2
    assert O.workspace_elements(True, 4, 9, 3, 5, 2) == 30
    assert O.workspace_elements(False, 2, 9, 2, 2, 1) == 4


# ---------------------------------------------------------- numerical pins
def _agree_case(rng, n, k, m, r):
    X, W, A, B, dY = (_rand(rng, *s) for s in [(n, k), (k, m), (k, r), (r, m), (n, m)])
    Y1 = O.forward(1, X, W, A, B)
    Y2 = O.forward(2, X, W, A, B)
    assert O.rel_fro(Y2, Y1) <= 1e-12
    ref = O.reference_backward(X, W, A, B, dY)
    for v in O.BWD_VARIANTS:
        got = O.backward(v, X, W, A, B, dY)
        for g, w in zip(got, ref):
            d = np.abs(g - w) / np.maximum(np.maximum(np.abs(g), np.abs(w)), 1e-12)
            # max-rel per S:66/S:251, guarded against cancellation to ~0
            assert np.all((d <= 1e-10) | (np.abs(g - w) <= 1e-12 * np.abs(w).max())), f"B{v}"


def test_variant_agreement_random():
    """Eq. 4: every bracketing agrees in fp64; 200 random shapes ≤ 64."""
    rng = np.random.default_rng(11)
    for _ in range(200):
        n, k, m = (int(x) for x in rng.integers(1, 65, 3))
        r = int(rng.integers(1, 17))
        _agree_case(rng, n, k, m, r)


def test_variant_agreement_medium():
    rng = np.random.default_rng(12)
    n, k, m, r = 512, 384, 384, 24
    X, W, A, B, dY = (_rand(rng, *s) for s in [(n, k), (k, m), (k, r), (r, m), (n, m)])
    ref = O.reference_backward(X, W, A, B, dY)
    for v in O.BWD_VARIANTS:
        for g, w in zip(O.backward(v, X, W, A, B, dY), ref):
            assert O.rel_fro(g, w) <= 1e-12


def test_finite_differences():
    """L = Σ Y∘G is affine in each single entry of X, A, B, so central differences
    with h = 1 are exact; also h = 1e-5 with the S:247 bound 1e-6."""
    rng = np.random.default_rng(3)
    cases = [(4, 3, 3, 2), (2, 1, 3, 1), (3, 2, 2, 2), (1, 4, 2, 1)] + [
        tuple(int(x) for x in rng.integers(1, 5, 3)) + (int(rng.integers(1, 3)),) for _ in range(20)]
    for (n, k, m, r) in cases:
        X, W, A, B, G = (_rand(rng, *s) for s in [(n, k), (k, m), (k, r), (r, m), (n, m)])
        L = lambda X_, A_, B_: float(np.sum(O.forward(1, X_, W, A_, B_) * G))
        for v in O.BWD_EXECUTABLE:
            dA, dB, dX = O.backward(v, X, W, A, B, G)
            for name, T, grad in (("X", X, dX), ("A", A, dA), ("B", B, dB)):
                for h, tol in ((1.0, 1e-10), (1e-5, 1e-6)):
                    fd = np.zeros_like(T)
                    for idx in np.ndindex(*T.shape):
                        Tp, Tm = T.copy(), T.copy()
                        Tp[idx] += h
                        Tm[idx] -= h
                        args_p = {"X": X, "A": A, "B": B, name: Tp}
                        args_m = {"X": X, "A": A, "B": B, name: Tm}
                        fd[idx] = (L(args_p["X"], args_p["A"], args_p["B"])
                                   - L(args_m["X"], args_m["A"], args_m["B"])) / (2 * h)
                    err = np.max(np.abs(fd - grad) / np.maximum(np.abs(grad), 1.0))
                    assert err <= tol, (v, name, h, err)


def test_torch_autograd_crosscheck():
    """Independent library routine: torch CPU fp64 autograd of Eq. 1."""
    rng = np.random.default_rng(21)
    for (n, k, m, r) in [(37, 29, 41, 5), (64, 64, 64, 8), (5, 80, 3, 2)]:
        X, W, A, B, dY = (_rand(rng, *s) for s in [(n, k), (k, m), (k, r), (r, m), (n, m)])
        tX, tA, tB = (torch.tensor(a, requires_grad=True) for a in (X, A, B))
        tW = torch.tensor(W)
        Y = tX @ tW + (tX @ tA) @ tB
        Y.backward(torch.tensor(dY))
        assert O.rel_fro(O.forward(1, X, W, A, B), Y.detach().numpy()) <= 1e-12
        for v in O.BWD_EXECUTABLE:
            dA, dB, dX = O.backward(v, X, W, A, B, dY)
            assert O.rel_fro(dA, tA.grad.numpy()) <= 1e-12
            assert O.rel_fro(dB, tB.grad.numpy()) <= 1e-12
            assert O.rel_fro(dX, tX.grad.numpy()) <= 1e-12


def test_special_cases():
    """A=0, B=0, X=0, dY=0, perturbing W."""
    rng = np.random.default_rng(4)
    n, k, m, r = 9, 7, 6, 3
    X, W, A, B, dY = (_rand(rng, *s) for s in [(n, k), (k, m), (k, r), (r, m), (n, m)])
    Z = np.zeros
    for v in O.FWD_VARIANTS:
        np.testing.assert_allclose(O.forward(v, X, W, Z((k, r)), B), X @ W, rtol=1e-13)
        np.testing.assert_allclose(O.forward(v, X, W, A, Z((r, m))), X @ W, rtol=1e-13)
        assert np.all(O.forward(v, Z((n, k)), W, A, B) == 0)
    for v in O.BWD_EXECUTABLE:
        dA, dB, dX = O.backward(v, X, W, A, B, Z((n, m)))
        assert np.all(dA == 0) and np.all(dB == 0) and np.all(dX == 0)
        dA, dB, dX = O.backward(v, Z((n, k)), W, A, B, dY)
        assert np.all(dA == 0) and np.all(dB == 0)
        np.testing.assert_allclose(dX, dY @ W.T + dY @ B.T @ A.T, rtol=1e-12)
        dA, dB, dX = O.backward(v, X, W, Z((k, r)), B, dY)
        assert np.all(dB == 0)
        np.testing.assert_allclose(dX, dY @ W.T, rtol=1e-12)
        dA, dB, dX = O.backward(v, X, W, A, Z((r, m)), dY)
        assert np.all(dA == 0)
        np.testing.assert_allclose(dX, dY @ W.T, rtol=1e-12)
    # dA, dB do not depend on W (Eq. 3 first two lines)
    for v in (1, 2, 3, 5):
        a1 = O.backward(v, X, W, A, B, dY)
        a2 = O.backward(v, X, W + 1.0, A, B, dY)
        np.testing.assert_array_equal(a1[0], a2[0])
        np.testing.assert_array_equal(a1[1], a2[1])


def test_rows_and_chunks_match_full():
    """Row-sampled Y/dX and chunked dA/dB equal the full evaluation."""
    rng = np.random.default_rng(8)
    n, k, m, r = 300, 40, 50, 6
    X, W, A, B, dY = (_rand(rng, *s) for s in [(n, k), (k, m), (k, r), (r, m), (n, m)])
    rows = np.array([0, 17, 128, 299])
    Y = O.forward(1, X, W, A, B)
    dA, dB, dX = O.reference_backward(X, W, A, B, dY)
    assert O.rel_fro(O.forward_rows(X[rows], W, A, B), Y[rows]) <= 1e-13
    assert O.rel_fro(O.dX_rows(dY[rows], W, A, B), dX[rows]) <= 1e-13
    gA, gB = O.adapter_grads(X, A, B, dY, row_chunk=64)
    assert O.rel_fro(gA, dA) <= 1e-13 and O.rel_fro(gB, dB) <= 1e-13


def test_rel_fro():
    assert O.rel_fro(np.ones((2, 2)), np.ones((2, 2))) == 0.0
    assert abs(O.rel_fro(np.array([[3.0, 4.0]]) * 1.1, np.array([[3.0, 4.0]])) - 0.1) < 1e-12
    assert O.rel_fro(np.zeros((1, 1)), np.zeros((1, 1))) == 0.0
