"""Pins of the quantized-weight oracle (oracle/quant.py) against the E4M3 definition and
plain arithmetic facts (no conversion library involved):

* decode: known codes of the OCP E4M3FN table (1.0 = 0x38, 448 = 0x7E, smallest
  subnormal 2^-9 = 0x01, smallest normal 2^-6 = 0x08, NaN = 0x7F/0xFF), 254 finite values,
  monotone over the positive codes, sign symmetry;
* encode: every finite value round-trips; midpoints between neighbours go to the even
  code; values beyond 448 saturate; the error of any encode is at most half a step;
* bf16 rounding: against torch's fp32 -> bf16 cast (an independent library routine);
* quantize / dequantize (R18, power-of-two column scales): the scale is the smallest power
  of two with amax/scale <= 448 (so the column max lands in (224, 448]) inside E5M2's
  [2^-16, 2^15]; the exponent rule against log2 and against brute force; W~ exact in bf16;
  relative error per element bounded by E4M3's half-ulp (2^-4 of the element's binade).
"""
import numpy as np
import torch

from oracle import quant as Q


def test_decode_known_codes():
    assert Q.e4m3_decode(0x38) == 1.0
    assert Q.e4m3_decode(0xB8) == -1.0
    assert Q.e4m3_decode(0x7E) == 448.0
    assert Q.e4m3_decode(0x01) == 2.0 ** -9
    assert Q.e4m3_decode(0x08) == 2.0 ** -6
    assert Q.e4m3_decode(0x07) == 7 / 8 * 2.0 ** -6
    assert np.isnan(Q.e4m3_decode(0x7F)) and np.isnan(Q.e4m3_decode(0xFF))
    t = Q.E4M3_TABLE
    assert np.sum(np.isfinite(t)) == 254
    pos = t[:0x7F]
    assert np.all(np.diff(pos) > 0)
    assert np.all(t[0x80:0xFF] == -t[:0x7F])


def test_encode_roundtrip_ties_saturation():
    codes = np.array([c for c in range(256) if np.isfinite(Q.E4M3_TABLE[c]) and c != 0x80])
    assert np.array_equal(Q.e4m3_encode(Q.E4M3_TABLE[codes]), codes.astype(np.uint8))
    assert Q.e4m3_encode(np.array([-0.0]))[0] == 0x80 and Q.e4m3_encode(np.array([0.0]))[0] == 0
    pos = Q.E4M3_TABLE[:0x7F]
    for c in range(0x7E):
        mid = (pos[c] + pos[c + 1]) / 2
        want = c if c % 2 == 0 else c + 1
        assert Q.e4m3_encode(np.array([mid]))[0] == want, c
        assert Q.e4m3_encode(np.array([-mid]))[0] == want | 0x80
    assert Q.e4m3_encode(np.array([1e6, -1e6, 449.0]))[0] == 0x7E
    rng = np.random.default_rng(3)
    x = rng.standard_normal(20000) * rng.choice([1e-3, 1.0, 100.0], 20000)
    x = np.clip(x, -448, 448).astype(np.float32).astype(np.float64)
    y = Q.E4M3_TABLE[Q.e4m3_encode(x)]
    step = np.where(np.abs(x) < 2.0 ** -6, 2.0 ** -9, 2.0 ** (np.floor(np.log2(np.maximum(np.abs(x), 1e-30))) - 3))
    assert np.all(np.abs(y - x) <= step / 2 + 1e-30)


def test_bf16_rne_matches_torch():
    rng = np.random.default_rng(4)
    x = (rng.standard_normal(100000) * 10.0 ** rng.uniform(-8, 8, 100000)).astype(np.float32)
    want = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(Q.bf16_rne(x), want)


def test_scale_exponent_rule():
    # brute force: the smallest e with amax / 2^e <= 448 (fp32 division), clamped
    rng = np.random.default_rng(6)
    amaxes = np.concatenate([rng.uniform(0, 1, 500) * 10.0 ** rng.integers(-8, 8, 500),
                             448.0 * 2.0 ** np.arange(-20, 20), [0.0, 1.0, 448.0, 449.0, 1e-30, 1e30]])
    for a in amaxes.astype(np.float32):
        e = Q.scale_exponent(float(a))
        if a == 0:
            assert e == 0
            continue
        x = np.float32(a) / np.float32(448.0)
        want = next(c for c in range(-200, 200) if np.float32(x) <= np.float32(2.0 ** c))
        assert e == min(max(want, -16), 15), (a, e, want)
    assert Q.scale_exponent(448.0) == 0 and Q.scale_exponent(449.0) == 1 and Q.scale_exponent(224.0) == -1


def test_quantize_dequantize_bounds():
    rng = np.random.default_rng(5)
    W = torch.from_numpy(rng.standard_normal((64, 48)) / 8).to(torch.bfloat16).double().numpy()
    W[:, 3] = 0.0
    W[:, 7] *= 1e-6  # a tiny column: exponent clamped at -16
    q, s = Q.quantize_w(W)
    assert q.dtype == np.uint8 and s.dtype == np.float32 and s[3] == 1.0
    e = np.log2(s.astype(np.float64))
    assert np.array_equal(e, np.round(e)) and e.min() >= -16 and e.max() <= 15  # powers of two
    Wd = Q.dequantize_w(q, s)
    assert np.array_equal(Q.bf16_rne(Wd.astype(np.float32)), Wd)  # W~ exact in bf16
    amax = np.abs(W).max(axis=0)
    for j in range(W.shape[1]):
        if amax[j] > 0 and e[j] > -16:
            i = np.argmax(np.abs(W[:, j]))
            assert 224.0 < abs(W[i, j]) / s[j] <= 448.0
            assert 224.0 <= abs(Q.E4M3_TABLE[q[i, j]]) <= 448.0
    # |W~ - W| <= half an E4M3 step of W/scale (relative 2^-4, or the subnormal step), times scale
    xs = np.abs(W) / s[None, :].astype(np.float64)
    step = np.where(xs < 2.0 ** -6, 2.0 ** -9, 2.0 ** (np.floor(np.log2(np.maximum(xs, 1e-30))) - 3))
    bound = step / 2 * s[None, :] + 1e-30
    assert np.all(np.abs(Wd - W) <= bound)
