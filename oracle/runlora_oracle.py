"""RunLoRA oracle: plain, slow, obviously-correct CPU fp64 implementation.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this module.
The product path (``paper_2312_03415_b200``) never imports it and shares no code
with it; the two meet only through the seeded inputs of ``synth`` (which holds none
of the method's arithmetic).

Citations ``P:n`` are lines of the paper's text (arXiv 2312.03415, PAPER.md);
``S:n`` lines of SPEC.md (used for interface/test ideas only).

Notation: the paper's b·s (tokens) is flattened to ``n`` (every Table 1 term
carries b·s), i = ``k`` (input dim), o = ``m`` (output dim), r = rank.
Layouts are the paper's: X[n,k], W[k,m] (Y = XW), A[k,r], B[r,m],
Y, dY[n,m], dX[n,k], dA[k,r], dB[r,m].

Every product goes through :class:`Counter.mm`, which counts 2·M·K·N FLOPs for an
(M×K)·(K×N) product and does not count matrix additions — the convention that
reproduces Table 1 exactly (reading R3).  The library
primitive used for a product step is ``numpy.matmul`` in float64.

Pins (what ties this file to the paper rather than to itself) live in
``tests/test_oracle.py``: worked integer/scalar examples (tests/golden/), the
Table 1 closed forms evaluated independently (SPEC numbers), the FLOP audit,
finite differences (exact for h=1 because the loss is affine per entry),
all-variant agreement (Eq. 4), torch-autograd of Eq. 1 as an independent library
routine, special cases, and the two dominance proofs.
Parity of every function here is pinned; none is "parity unpinned".
"""
from __future__ import annotations

import numpy as np

FWD_VARIANTS = (1, 2)
BWD_VARIANTS = (1, 2, 3, 4, 5, 6, 7, 8)
BWD_EXECUTABLE = (1, 2, 3, 4, 5)         # P:96-98 "we implement only first five"


class Counter:
    """Counting matrix product: the only way the oracle multiplies matrices."""

    def __init__(self):
        self.flops = 0

    def mm(self, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        assert a.ndim == 2 and b.ndim == 2 and a.shape[1] == b.shape[0], (a.shape, b.shape)
        self.flops += 2 * a.shape[0] * a.shape[1] * b.shape[1]
        return np.matmul(a, b)


def _f64(*xs):
    return [np.asarray(x, dtype=np.float64) for x in xs]


# ---------------------------------------------------------------- forward (§2)
def forward(v: int, X, W, A, B, ctr: Counter | None = None) -> np.ndarray:
    """Major forward variants.

    v=1: Y = (XW) + ((XA)B)      (Eq. 1; item 1)
    v=2: Y = X(W + AB)           (Eq. 2; item 2)
    Nothing is saved for the backward."""
    X, W, A, B = _f64(X, W, A, B)
    c = ctr if ctr is not None else Counter()
    if v == 1:
        return c.mm(X, W) + c.mm(c.mm(X, A), B)
    if v == 2:
        return c.mm(X, W + c.mm(A, B))
    raise ValueError(f"forward variant {v} does not exist (P:62-64)")


# --------------------------------------------------------------- backward (§2)
def backward(v: int, X, W, A, B, dY, ctr: Counter | None = None):
    """Backward variants; returns (dA, dB, dX).

    v=1..5 follow Algorithms 1-5 line by line.  v=6..8 follow the
    bracketings enumerated at P:91-93; the paper does not execute them,
    the oracle evaluates them only for the FLOP audit and agreement tests.
    Only X, W, A, B, dY are inputs: nothing from a forward is reused."""
    X, W, A, B, dY = _f64(X, W, A, B, dY)
    c = ctr if ctr is not None else Counter()
    T = np.transpose
    if v == 1:                          # Alg. 1
        Z1 = c.mm(dY, T(B))
        Z2 = c.mm(X, A)
        dA = c.mm(T(X), Z1)
        dB = c.mm(T(Z2), dY)
        dX = c.mm(dY, T(W)) + c.mm(Z1, T(A))
    elif v == 2:                        # Alg. 2
        Z1 = c.mm(dY, T(B))
        Z2 = c.mm(T(X), dY)
        dA = c.mm(T(X), Z1)
        dB = c.mm(T(A), Z2)
        dX = c.mm(dY, T(W)) + c.mm(Z1, T(A))
    elif v == 3:                        # Alg. 3
        Z1 = c.mm(dY, T(B))
        Z2 = c.mm(T(X), dY)
        dA = c.mm(Z2, T(B))
        dB = c.mm(T(A), Z2)
        dX = c.mm(dY, T(W)) + c.mm(Z1, T(A))
    elif v == 4:                        # Alg. 4
        Z1 = W + c.mm(A, B)
        Z2 = c.mm(T(X), dY)
        dA = c.mm(Z2, T(B))
        dB = c.mm(T(A), Z2)
        dX = c.mm(dY, T(Z1))
    elif v == 5:                        # Alg. 5
        Z1 = c.mm(dY, T(B))
        Z2 = c.mm(X, A)
        Z3 = W + c.mm(A, B)
        dA = c.mm(T(X), Z1)
        dB = c.mm(T(Z2), dY)
        dX = c.mm(dY, T(Z3))
    elif v == 6:                        # item 6
        dA = c.mm(c.mm(T(X), dY), T(B))
        dB = c.mm(c.mm(T(A), T(X)), dY)
        dX = c.mm(dY, T(W)) + c.mm(c.mm(dY, T(B)), T(A))
    elif v == 7:                        # item 7
        dA = c.mm(c.mm(T(X), dY), T(B))
        dB = c.mm(c.mm(T(A), T(X)), dY)
        dX = c.mm(dY, T(W) + c.mm(T(B), T(A)))
    elif v == 8:                        # item 8
        dA = c.mm(T(X), c.mm(dY, T(B)))
        dB = c.mm(T(A), c.mm(T(X), dY))
        dX = c.mm(dY, T(W) + c.mm(T(B), T(A)))
    else:
        raise ValueError(f"backward variant {v} does not exist (P:84-94)")
    return dA, dB, dX


def reference_backward(X, W, A, B, dY):
    """Eq. 3 in one fixed association order:
    dA = Xᵀ(dY Bᵀ), dB = Aᵀ(Xᵀ dY), dX = dY Wᵀ + (dY Bᵀ) Aᵀ."""
    X, W, A, B, dY = _f64(X, W, A, B, dY)
    T = np.transpose
    dA = T(X) @ (dY @ T(B))
    dB = T(A) @ (T(X) @ dY)
    dX = dY @ T(W) + (dY @ T(B)) @ T(A)
    return dA, dB, dX


# ------------------------------------------------------- large-shape evaluation
def forward_rows(X_rows, W, A, B) -> np.ndarray:
    """Rows of Y = XW + (XA)B for a subset of token rows (Eq. 1 is row-wise in X)."""
    X_rows, W, A, B = _f64(X_rows, W, A, B)
    return X_rows @ W + (X_rows @ A) @ B


def dX_rows(dY_rows, W, A, B) -> np.ndarray:
    """Rows of dX = dY Wᵀ + (dY Bᵀ) Aᵀ (Eq. 3 third line is row-wise in dY)."""
    dY_rows, W, A, B = _f64(dY_rows, W, A, B)
    return dY_rows @ W.T + (dY_rows @ B.T) @ A.T


def adapter_grads(X, A, B, dY, row_chunk: int = 16384):
    """Full dA, dB of Eq. 3 via dA = Xᵀ(dY Bᵀ), dB = (XA)ᵀ dY — the n-linear
    association (Alg. 1 lines P:103-106), accumulated over token-row chunks so the
    fp64 copies of X and dY never need to be materialised whole."""
    A, B = _f64(A, B)
    k, r = A.shape
    m = B.shape[1]
    dA = np.zeros((k, r))
    dB = np.zeros((r, m))
    n = X.shape[0]
    for t0 in range(0, n, row_chunk):
        Xc = np.asarray(X[t0:t0 + row_chunk], dtype=np.float64)
        dYc = np.asarray(dY[t0:t0 + row_chunk], dtype=np.float64)
        dA += Xc.T @ (dYc @ B.T)
        dB += (Xc @ A).T @ dYc
    return dA, dB


# --------------------------------------------------------- cost model (Table 1)
def flops_forward(v: int, n: int, k: int, m: int, r: int) -> int:
    """Table 1 rows forward1/forward2, exact integers; n = b·s, i = k, o = m."""
    i, o = k, m
    if v == 1:
        return 2 * n * (i * o + r * i + o * r)
    if v == 2:
        return 2 * (i * o * r + n * o * i)
    raise ValueError(v)


def flops_backward(v: int, n: int, k: int, m: int, r: int) -> int:
    """Table 1 rows backward1..8 as printed, exact integers."""
    i, o = k, m
    if v == 1:
        return 2 * n * (2 * o * r + 3 * i * r + o * i)
    if v == 2:
        return 2 * n * (o * r + 2 * i * r + 2 * i * o) + 2 * i * o * r
    if v == 3:
        return 2 * n * (2 * i * o + o * r + i * r) + 4 * i * r * o
    if v == 4:
        return 2 * (2 * n * i * o + 3 * i * o * r)
    if v == 5:
        return 2 * n * (2 * o * r + 2 * i * r + o * i) + 2 * i * o * r
    if v == 6:
        return 2 * n * (2 * o * r + 2 * i * r + 2 * o * i) + 4 * i * o * r
    if v in (7, 8):
        return 2 * n * (o * r + i * r + 2 * o * i) + 4 * i * o * r
    raise ValueError(v)


def param_reduction(k: int, m: int, r: int) -> bool:
    """Eq. 5: r(i + o) < io, strict."""
    return r * (k + m) < k * m


def select_by_flops(n: int, k: int, m: int, r: int):
    """FLOP criterion (P:5): argmin over {F1,F2} and over the executable
    {B1..B5}; ties go to the lowest variant index (R5)."""
    f = min(FWD_VARIANTS, key=lambda v: (flops_forward(v, n, k, m, r), v))
    b = min(BWD_EXECUTABLE, key=lambda v: (flops_backward(v, n, k, m, r), v))
    return f, b


def baseline_flops(n: int, k: int, m: int, r: int):
    """Default chain (Eq. 1 + autograd) modelled as forward1 that caches XA
    and backward1 that reuses it: (F1, B1 − 2·n·k·r)."""
    return flops_forward(1, n, k, m, r), flops_backward(1, n, k, m, r) - 2 * n * k * r


def workspace_elements(is_backward: bool, v: int, n: int, k: int, m: int, r: int) -> int:
    """Temporaries of each executable variant: the Z's of Alg. 1-5 and
    the XA / W+AB of the forwards."""
    if not is_backward:
        return {1: n * r, 2: k * m}[v]
    return {1: 2 * n * r, 2: n * r + k * m, 3: n * r + k * m, 4: 2 * k * m,
            5: 2 * n * r + k * m}[v]


def rel_fro(got, want) -> float:
    """Relative Frobenius error ‖G − O‖_F / ‖O‖_F (BASELINE.json tolerance metric)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    den = np.linalg.norm(want)
    num = np.linalg.norm(got - want)
    if den == 0.0:
        return float(num)
    return float(num / den)
