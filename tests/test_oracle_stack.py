"""Pins of the C5 stack oracle (oracle/stack.py) against things other than itself:

* torch fp64 autograd of the same dataflow (reading R15: weightless RMS
  pre-norm residual blocks), written here with plain torch ops — an independent
  library routine for the chain rule, the RMS normalisation's derivative included;
* central finite differences of L = Σ Y ∘ G on a tiny stack (the loss is smooth but
  not affine in an entry because of g ⊙ u, so h = 1e-6 with a 1e-6 bound);
* DP linearity: the sum of shard gradients equals the full-batch gradients.
"""
import numpy as np
import torch

from oracle import stack as S


def _layers(rng, nl, d, f, r):
    dims = {"gate": (d, f), "up": (d, f), "down": (f, d)}
    out = []
    for _ in range(nl):
        L = {}
        for name in S.LINEARS:
            k, m = dims.get(name, (d, d))
            L[name] = {"W": rng.standard_normal((k, m)) / np.sqrt(k), "A": rng.standard_normal((k, r)) / np.sqrt(k),
                       "B": rng.standard_normal((r, m)) / np.sqrt(r)}
        out.append(L)
    return out


def _torch_stack(x, layers):
    """The same dataflow in torch (fp64 autograd)."""
    params = []
    xt = torch.tensor(x, requires_grad=True)
    h = xt

    def lin(z, p):
        W = torch.tensor(p["W"])
        A = torch.tensor(p["A"], requires_grad=True)
        B = torch.tensor(p["B"], requires_grad=True)
        params.append((A, B))
        return z @ W + (z @ A) @ B

    def rms(z):
        return z / torch.sqrt((z * z).mean(dim=1, keepdim=True) + 1e-6)

    for L in layers:
        n1 = rms(h)
        a = lin(n1, L["q"]) + lin(n1, L["k"]) + lin(n1, L["v"])
        x1 = h + lin(a, L["o"])
        n2 = rms(x1)
        g = lin(n2, L["gate"])
        u = lin(n2, L["up"])
        h = x1 + lin(g * u, L["down"])
    return xt, h, params


def test_stack_matches_torch_autograd():
    rng = np.random.default_rng(14)
    n, d, f, r, nl = 5, 6, 10, 3, 3
    layers = _layers(rng, nl, d, f, r)
    x = rng.standard_normal((n, d))
    dy = rng.standard_normal((n, d))
    y, cache = S.stack_forward(x, layers)
    dx, grads = S.stack_backward(dy, layers, cache)
    xt, yt, params = _torch_stack(x, layers)
    yt.backward(torch.tensor(dy))
    assert np.allclose(y, yt.detach().numpy(), rtol=1e-12, atol=1e-12)
    assert np.allclose(dx, xt.grad.numpy(), rtol=1e-11, atol=1e-11)
    i = 0
    for li in range(nl):
        for name in ("q", "k", "v", "o", "gate", "up", "down"):  # creation order in _torch_stack
            A, B = params[i]
            i += 1
            gA, gB = grads[li][name]
            assert np.allclose(gA, A.grad.numpy(), rtol=1e-11, atol=1e-11), (li, name)
            assert np.allclose(gB, B.grad.numpy(), rtol=1e-11, atol=1e-11), (li, name)


def test_stack_finite_differences():
    rng = np.random.default_rng(15)
    n, d, f, r, nl = 2, 3, 4, 2, 2
    layers = _layers(rng, nl, d, f, r)
    x = rng.standard_normal((n, d))
    G = rng.standard_normal((n, d))
    _, cache = S.stack_forward(x, layers)
    dx, grads = S.stack_backward(G, layers, cache)

    def loss():
        return float(np.sum(S.stack_forward(x, layers)[0] * G))

    h = 1e-6
    for li in range(nl):
        for name in ("q", "o", "gate", "down"):
            for key, gi in (("A", 0), ("B", 1)):
                M = layers[li][name][key]
                idx = tuple(rng.integers(0, s) for s in M.shape)
                old = M[idx]
                M[idx] = old + h
                lp = loss()
                M[idx] = old - h
                lm = loss()
                M[idx] = old
                fd = (lp - lm) / (2 * h)
                an = grads[li][name][gi][idx]
                assert abs(fd - an) <= 1e-6 * max(1.0, abs(an)), (li, name, key, fd, an)
    for idx in [(0, 0), (1, 2)]:
        old = x[idx]
        x[idx] = old + h
        lp = loss()
        x[idx] = old - h
        lm = loss()
        x[idx] = old
        assert abs((lp - lm) / (2 * h) - dx[idx]) <= 1e-6 * max(1.0, abs(dx[idx]))


def test_stack_dp_linearity():
    """Adapter grads are sums over tokens: shard grads add up to the full-batch grads."""
    rng = np.random.default_rng(16)
    n, d, f, r = 8, 4, 6, 2
    layers = _layers(rng, 2, d, f, r)
    x = rng.standard_normal((n, d))
    dy = rng.standard_normal((n, d))
    _, full = S.stack_backward(dy, layers, S.stack_forward(x, layers)[1])
    acc = None
    for lo, hi in ((0, 3), (3, 8)):
        _, g = S.stack_backward(dy[lo:hi], layers, S.stack_forward(x[lo:hi], layers)[1])
        acc = g if acc is None else [{k: (a[k][0] + b[k][0], a[k][1] + b[k][1]) for k in a} for a, b in zip(acc, g)]
    for a, b in zip(acc, full):
        for k in a:
            assert np.allclose(a[k][0], b[k][0], rtol=1e-12, atol=1e-12)
            assert np.allclose(a[k][1], b[k][1], rtol=1e-12, atol=1e-12)
