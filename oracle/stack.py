"""CPU fp64 oracle of the C5 stack — TEST INFRASTRUCTURE ONLY (same rules as
runlora_oracle.py: only tests/ and bench.py's baseline legs may use it).

BASELINE.json configs[4] gives the C5 stack's shapes only ("32-layer stack of
LoRA-adapted linears with Llama-7B projection shapes per layer (q, k, v, o at
4096x4096; gate and up at 4096x11008; down at 11008x4096), no attention").  The
dataflow is DESIGN.md reading R15: Llama's pre-norm residual blocks with the
attention and the SiLU removed and a weightless RMS normalisation (without it the
gate product squares the activations' scale every layer and a 32-layer stack of
random weights overflows bf16):

    h = rms(x);   a = L_q(h) + L_k(h) + L_v(h);   x1 = x + L_o(a)
    h2 = rms(x1); x2 = x1 + L_down(L_gate(h2) ⊙ L_up(h2))
    rms(z) = z / sqrt(mean(z², row) + eps),  eps = 1e-6

Every L is one LoRA-adapted linear, Y = XW + (XA)B (Eq. 1), whose
gradients are Eq. 3 — both taken from runlora_oracle (``forward`` with
variant 1, ``reference_backward``).  The backward seeds the stack output with a
given dY (there is no loss) and applies the chain rule through the glue above.

Pins: tests/test_oracle_stack.py checks this file against torch fp64 autograd of
the same dataflow written with torch ops (an independent library routine) and
against central finite differences on a tiny stack.
"""
from __future__ import annotations

import numpy as np

from .runlora_oracle import forward, reference_backward

LINEARS = ("q", "k", "v", "o", "gate", "up", "down")


EPS = 1e-6


def _lin(x, p):
    return forward(1, x, p["W"], p["A"], p["B"])  # Eq. 1


def rms(z):
    """Row-wise RMS normalisation and the scale s = (mean(z²) + eps)^(-1/2) per row."""
    s = 1.0 / np.sqrt(np.mean(z * z, axis=1, keepdims=True) + EPS)
    return z * s, s


def rms_backward(z, s, dy):
    """d/dz of y = z·s(z): dz = s·dy - z·s³·mean(z ⊙ dy, row)."""
    return s * dy - z * (s ** 3) * np.mean(z * dy, axis=1, keepdims=True)


def stack_forward(x, layers):
    """Stack output and the per-layer intermediates the backward needs (fp64)."""
    x = np.asarray(x, dtype=np.float64)
    cache = []
    for L in layers:
        h, s1 = rms(x)
        a = _lin(h, L["q"]) + _lin(h, L["k"]) + _lin(h, L["v"])
        x1 = x + _lin(a, L["o"])
        h2, s2 = rms(x1)
        g = _lin(h2, L["gate"])
        u = _lin(h2, L["up"])
        p = g * u
        cache.append({"x": x, "h": h, "s1": s1, "a": a, "x1": x1, "h2": h2, "s2": s2, "g": g, "u": u, "p": p})
        x = x1 + _lin(p, L["down"])
    return x, cache


def stack_backward(dy, layers, cache):
    """(dX of the stack input, [{name: (dA, dB)}] per layer) for output gradient dy."""
    dy = np.asarray(dy, dtype=np.float64)
    grads = [None] * len(layers)
    for li in range(len(layers) - 1, -1, -1):
        L, c, G = layers[li], cache[li], {}
        # x2 = x1 + L_down(p)
        dA, dB, dp = reference_backward(c["p"], L["down"]["W"], L["down"]["A"], L["down"]["B"], dy)
        G["down"] = (dA, dB)
        dg, du = dp * c["u"], dp * c["g"]  # p = g ⊙ u
        dA, dB, dh2_g = reference_backward(c["h2"], L["gate"]["W"], L["gate"]["A"], L["gate"]["B"], dg)
        G["gate"] = (dA, dB)
        dA, dB, dh2_u = reference_backward(c["h2"], L["up"]["W"], L["up"]["A"], L["up"]["B"], du)
        G["up"] = (dA, dB)
        dx1 = dy + rms_backward(c["x1"], c["s2"], dh2_g + dh2_u)  # h2 = rms(x1)
        # x1 = x + L_o(a)
        dA, dB, da = reference_backward(c["a"], L["o"]["W"], L["o"]["A"], L["o"]["B"], dx1)
        G["o"] = (dA, dB)
        dh = 0.0
        for name in ("q", "k", "v"):  # a = L_q(h) + L_k(h) + L_v(h)
            dA, dB, dxh = reference_backward(c["h"], L[name]["W"], L[name]["A"], L[name]["B"], da)
            G[name] = (dA, dB)
            dh = dh + dxh
        grads[li] = G
        dy = dx1 + rms_backward(c["x"], c["s1"], dh)  # h = rms(x)
    return dy, grads
