"""CPU oracle of the quantized frozen weight — TEST INFRASTRUCTURE ONLY (same rules as
runlora_oracle.py: only tests/ and bench.py's baseline legs may use it).

PAPER.md P:20: "We also provide a functionality to work with quantized model weights to
fine-tune models in fashion of QLoRA" — no format is given.  The
format chosen (reading R18) is FP8 E4M3 with one fp32 scale per output column:

    scale[j] = max_i |W[i, j]| / 448   (1 when the column is all zero)
    Wq[i, j] = e4m3_rne_satfinite(W[i, j] / scale[j])      (fp32 division, then RNE)
    W~[i, j] = bf16_rne(fp32(e4m3(Wq[i, j]) · scale[j]))   (the bf16 W the hot path uses)

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


def quantize_w(W) -> tuple[np.ndarray, np.ndarray]:
    """(Wq bytes [k, m], scale fp32 [m]) of a bf16-valued W [k, m] (reading R18)."""
    W32 = np.asarray(W, dtype=np.float32)
    amax = np.max(np.abs(W32), axis=0)
    scale = np.where(amax > 0, amax / np.float32(E4M3_MAX), np.float32(1.0)).astype(np.float32)
    q = e4m3_encode((W32 / scale[None, :]).astype(np.float32))
    return q, scale


def dequantize_w(Wq, scale) -> np.ndarray:
    """W~ = bf16(fp32(e4m3(Wq)) · scale) as fp64 values [k, m]."""
    v = E4M3_TABLE[np.asarray(Wq, dtype=np.uint8)].astype(np.float32)
    return bf16_rne(v * np.asarray(scale, dtype=np.float32)[None, :])
