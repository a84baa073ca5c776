"""CPU oracle of the quantized frozen weight — TEST INFRASTRUCTURE ONLY (same rules as
runlora_oracle.py: only tests/ and bench.py's baseline legs may use it).

PAPER.md P:20: "We also provide a functionality to work with quantized model weights to
fine-tune models in fashion of QLoRA" — no format is given.  The
format chosen (reading R18, revised in round 2) is FP8 E4M3 with one power-of-two
scale per output column (an E8M0-style exponent, as in the OCP MX formats):

    e[j]     = clamp(ceil(log2(amax_j / 448)), -16, 15),  amax_j = max_i |W[i, j]|
               (e[j] = 0 when the column is all zero; amax_j / 448 is an fp32 division)
    scale[j] = 2^e[j]
    Wq[i, j] = e4m3_rne_satfinite(W[i, j] / scale[j])      (exact division, then RNE)
    W~[i, j] = e4m3(Wq[i, j]) · scale[j]                   (exact: 4 significant bits, so
                                                            also exact in bf16)
Round 1 used scale = amax/448 (any fp32) and W~ = bf16_rne(e4m3 · scale); the power of two
makes W~ exact, so the tensor cores can apply the scale as an E5M2 diagonal matrix (the
clamp is E5M2's range of powers of two, 2^-16 .. 2^15).

E4M3 here is the OCP "E4M3FN" encoding: 1 sign, 4 exponent (bias 7), 3 mantissa bits;
exponent field 0 = subnormals (m/8 · 2^-6); S.1111.111 = NaN; no infinities; max 448.
Everything below is written from that definition (bit fields, exhaustive nearest search)
rather than from any conversion routine, and pinned in tests/test_oracle_quant.py.
"""
from __future__ import annotations

import numpy as np

E4M3_MAX = 448.0


def e4m3_decode(code: int) -> float:
    """Value of one E4M3FN byte (NaN for S.1111.111)."""
    s = -1.0 if code & 0x80 else 1.0
    e = (code >> 3) & 0xF
    mant = code & 0x7
    if e == 0xF and mant == 0x7:
        return float("nan")
    if e == 0:
        return s * (mant / 8.0) * 2.0 ** -6
    return s * (1.0 + mant / 8.0) * 2.0 ** (e - 7)


E4M3_TABLE = np.array([e4m3_decode(c) for c in range(256)], dtype=np.float64)


def e4m3_encode(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even onto the finite E4M3FN values, saturating at ±448 (x: fp32
    values, exactly representable in fp64).  Ties go to the code with an even mantissa; the
    sign bit is kept, so values that round to zero from below give -0 (0x80)."""
    x = np.asarray(x, dtype=np.float64)
    codes = np.arange(256)
    finite = ~np.isnan(E4M3_TABLE)
    pos = codes[finite & (codes < 0x80)]          # +0 .. +448, increasing value
    vals = E4M3_TABLE[pos]
    a = np.minimum(np.abs(x), E4M3_MAX)
    idx = np.searchsorted(vals, a)                 # first value >= a
    idx = np.clip(idx, 1, len(vals) - 1)
    lo, hi = vals[idx - 1], vals[idx]
    d_lo, d_hi = a - lo, hi - a
    pick_hi = (d_hi < d_lo) | ((d_hi == d_lo) & ((pos[idx] & 1) == 0))
    out = np.where(pick_hi, pos[idx], pos[idx - 1])
    out = np.where(a == 0, 0, out)
    return (out | np.where(np.signbit(x), 0x80, 0)).astype(np.uint8)  # the sign survives (-0 = 0x80)


def bf16_rne(x32: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 (round to nearest even on the upper 16 bits), returned as fp64 values."""
    b = np.asarray(x32, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounded = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16) << 16
    return rounded.astype(np.uint32).view(np.float32).astype(np.float64)


SCALE_EXP_MIN, SCALE_EXP_MAX = -16, 15


def scale_exponent(amax: float) -> int:
    """e = ceil(log2(fp32(amax / 448))) clamped to [-16, 15]; 0 for amax = 0 (reading R18)."""
    if amax == 0:
        return 0
    x = float(np.float32(np.float32(amax) / np.float32(E4M3_MAX)))
    m, e = np.frexp(x)                   # x = m · 2^e, 0.5 <= m < 1
    c = int(e) - 1 if m == 0.5 else int(e)  # ceil(log2 x): exact powers of two stay
    return min(max(c, SCALE_EXP_MIN), SCALE_EXP_MAX)


def quantize_w(W) -> tuple[np.ndarray, np.ndarray]:
    """(Wq bytes [k, m], scale fp32 [m], powers of two) of a bf16-valued W [k, m] (R18)."""
    W32 = np.asarray(W, dtype=np.float32)
    amax = np.max(np.abs(W32), axis=0)
    scale = np.array([2.0 ** scale_exponent(a) for a in amax], dtype=np.float32)
    q = e4m3_encode((W32.astype(np.float64) / scale[None, :].astype(np.float64)).astype(np.float32))
    return q, scale


def dequantize_w(Wq, scale) -> np.ndarray:
    """W~ = e4m3(Wq) · scale as fp64 values [k, m] (exact)."""
    v = E4M3_TABLE[np.asarray(Wq, dtype=np.uint8)]
    return v * np.asarray(scale, dtype=np.float64)[None, :]
