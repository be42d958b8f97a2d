"""Pins for oracle/quant.py and the synthetic quantiser in paper_2508_15601_b200/synth.py."""

import json
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle.quant import dequant_f64, dequant_rounded
from oracle.numerics import round_bf16, round_fp16

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "dequant_examples.json")))


def _one(q, s, z, group=64):
    """Place one (q, s, z) at element (0, 0) of a minimal [group][128] problem."""
    qq = np.zeros((group, 128), dtype=np.uint8)
    ss = np.ones((1, 128), dtype=np.float16)
    zz = np.zeros((1, 128), dtype=np.float16)
    qq[0, 0], ss[0, 0], zz[0, 0] = q, s, z
    return qq, ss, zz


@pytest.mark.parametrize("ex", GOLDEN["spec_dequant"])
def test_spec_dequant_examples(ex):
    qq, ss, zz = _one(ex["q"], ex["s"], ex["z"])
    assert dequant_f64(qq, ss, zz, 64)[0, 0] == ex["out"]
    for dt in ("bf16", "fp16"):
        assert dequant_rounded(qq, ss, zz, 64, dt)[0, 0] == ex["out"]


@pytest.mark.parametrize("ex", GOLDEN["rounding"])
def test_rounding_sequence_worked_example(ex):
    qq, ss, zz = _one(ex["q"], ex["s"], ex["z"])
    assert float(np.float16(ex["s"])) == ex["s"]
    assert dequant_f64(qq, ss, zz, 64)[0, 0] == ex["exact"]
    assert dequant_rounded(qq, ss, zz, 64, "bf16")[0, 0] == ex["bf16"]
    assert dequant_rounded(qq, ss, zz, 64, "fp16")[0, 0] == ex["fp16"]


def test_dequant_exact_rationals():
    """Exact rational (q - z) * s on random fp16 scales equals the float64 evaluation."""
    rng = np.random.default_rng(2)
    K, N, g = 128, 128, 64
    q = rng.integers(0, 16, size=(K, N), dtype=np.uint8)
    s = rng.uniform(1e-4, 2.0, size=(K // g, N)).astype(np.float16)
    z = rng.integers(0, 16, size=(K // g, N)).astype(np.float16)
    W = dequant_f64(q, s, z, g)
    for _ in range(300):
        k, n = int(rng.integers(K)), int(rng.integers(N))
        exact = (Fraction(int(q[k, n])) - Fraction(float(z[k // g, n]))) * Fraction(float(s[k // g, n]))
        assert Fraction(W[k, n]) == exact


def test_group_boundaries():
    """k = g*group ... (g+1)*group-1 uses row g of s and z, for group 64 and 128."""
    for g in (64, 128):
        K, N = 256, 128
        q = np.full((K, N), 5, dtype=np.uint8)
        s = np.arange(1, K // g + 1, dtype=np.float16)[:, None].repeat(N, 1)
        z = np.zeros((K // g, N), dtype=np.float16)
        W = dequant_f64(q, s, z, g)
        for k in range(K):
            assert W[k, 0] == 5 * (k // g + 1)


def test_high_nibble_ignored():
    q = np.full((64, 128), 0xA3, dtype=np.uint8)
    s = np.ones((1, 128), dtype=np.float16)
    z = np.zeros((1, 128), dtype=np.float16)
    assert np.all(dequant_f64(q, s, z, 64) == 3.0)


def test_rounded_closed_forms_exhaustive_codes():
    """For integer zeros: bf16 sequence == RNE_bf16(RNE_bf16(s)*(q-z)); fp16 sequence ==
    RNE_fp16((q-z)*s).  All 16 x 16 (q, z) pairs x 2000 random +- scales."""
    rng = np.random.default_rng(4)
    bits = rng.integers(0, 0x7C00, size=2000).astype(np.uint16)
    sv = bits.view(np.float16).astype(np.float64) * np.where(rng.random(2000) < 0.5, -1, 1)
    qv, zv = np.meshgrid(np.arange(16), np.arange(16), indexing="ij")
    qv, zv = qv.ravel(), zv.ravel()
    K = 64
    for s in sv[:200]:
        q = np.zeros((K, 256), dtype=np.uint8)
        z = np.zeros((1, 256), dtype=np.float16)
        q[0, :] = qv
        z[0, :] = zv
        ss = np.full((1, 256), s, dtype=np.float16)
        got_b = dequant_rounded(q, ss, z, K, "bf16")[0]
        got_h = dequant_rounded(q, ss, z, K, "fp16")[0]
        d = (qv - zv).astype(np.float64)
        np.testing.assert_array_equal(got_b, round_bf16(round_bf16(s) * d))
        np.testing.assert_array_equal(got_h, round_fp16(d * s))
        # sign of zero: (q - z) * s with q == z is +0 * s
        zero = qv == zv
        assert np.array_equal(np.signbit(got_h[zero]), np.full(zero.sum(), s < 0))


@pytest.mark.parametrize("ex", GOLDEN["spec_quantize"])
def test_synth_quantizer_spec_examples(ex):
    from paper_2508_15601_b200.synth import quantize_minmax
    W = np.array(ex["values"], dtype=np.float32)[:, None]
    q, s, z = quantize_minmax(W, len(ex["values"]))
    assert float(s[0, 0]) == ex["scale"]
    assert float(z[0, 0]) == ex["zp"]
    assert q[:, 0].tolist() == ex["codes"]
    # dequantize returns the values (exact zeros for the all-zero group)
    Wd = dequant_f64(q, s, z, len(ex["values"]))
    assert np.array_equal(Wd[:, 0], np.array(ex["values"], dtype=np.float64))


def test_synth_roundtrip_error_bound():
    """|dequant(quantize(w)) - w| <= scale/2 (+ fp16 slack of the scale)."""
    from paper_2508_15601_b200.synth import quantize_minmax
    rng = np.random.default_rng(8)
    W = rng.normal(0, 0.02, size=(512, 256)).astype(np.float32)
    q, s, z = quantize_minmax(W, 128)
    Wd = dequant_f64(q, s, z, 128)
    smax = np.repeat(s.astype(np.float64), 128, axis=0)
    # scale is rounded to fp16, so the grid can stretch by up to 2^-11 relative over 15 steps
    assert np.all(np.abs(Wd - W) <= smax * (0.5 + 15 * 2.0 ** -10) + 1e-12)
    assert q.max() <= 15 and np.all(z.astype(np.float64) == np.rint(z.astype(np.float64)))
