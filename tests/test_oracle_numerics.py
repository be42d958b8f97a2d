"""Pins for oracle/numerics.py (RNE to bf16 / fp16) against independent implementations."""

import numpy as np
import pytest

from oracle.numerics import round_bf16, round_fp16, bf16_bits, fp16_bits, bf16_from_bits


def _bf16_bittrick(x32):
    """Independent float32 -> bf16 RNE via the integer rounding-bias trick."""
    b = np.asarray(x32, dtype=np.float32).view(np.uint32).astype(np.uint64)
    bias = 0x7FFF + ((b >> 16) & 1)
    return (((b + bias) >> 16) & 0xFFFF).astype(np.uint16)


def test_fp16_matches_numpy_cast_random():
    rng = np.random.default_rng(0)
    x = np.concatenate([
        rng.normal(0, 1, 20000),
        rng.normal(0, 1e-5, 20000),          # subnormal range of fp16
        rng.normal(0, 3e4, 20000),           # near overflow
        np.ldexp(rng.uniform(-1, 1, 20000), rng.integers(-30, 17, 20000)),
    ])
    ref = x.astype(np.float16).astype(np.float64)
    got = round_fp16(x)
    assert np.array_equal(np.isinf(ref), np.isinf(got))
    fin = np.isfinite(ref)
    assert np.array_equal(got[fin], ref[fin])


def test_fp16_ties_and_spec_examples():
    # 1.0 -> 1.0; 2049 -> 2048 (tie to even); 65520 -> +inf
    assert round_fp16(1.0) == 1.0
    assert round_fp16(2049.0) == 2048.0
    assert round_fp16(2051.0) == 2052.0
    assert np.isinf(round_fp16(65520.0)) and round_fp16(65520.0) > 0
    assert round_fp16(65519.0) == 65504.0
    assert round_fp16(-65520.0) == -np.inf
    # ties crafted at the midpoints of every binade agree with numpy's correctly rounded cast
    mids = []
    for e in range(-24, 16):
        for m in range(0, 1024, 37):
            lo = np.ldexp(1024 + m, e - 10)
            mids.append(lo + np.ldexp(1.0, e - 11))
    mids = np.array(mids)
    fin = np.isfinite(mids.astype(np.float16))
    assert np.array_equal(round_fp16(mids)[fin], mids.astype(np.float16).astype(np.float64)[fin])


def test_bf16_matches_bittrick_and_torch():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(1)
    x32 = np.concatenate([
        rng.normal(0, 1, 50000),
        np.ldexp(rng.uniform(-2, 2, 50000), rng.integers(-120, 120, 50000)),
    ]).astype(np.float32)
    got_bits = bf16_bits(round_bf16(x32.astype(np.float64)))
    assert np.array_equal(got_bits, _bf16_bittrick(x32))
    tb = torch.from_numpy(x32).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got_bits, tb)


def test_bf16_ties():
    u = 2.0 ** -7  # bf16 ulp at 1
    assert round_bf16(1 + u / 2) == 1.0                # tie -> even mantissa 0
    assert round_bf16(1 + 3 * u / 2) == 1 + 2 * u      # tie -> even mantissa 2
    assert round_bf16(1 + u / 2 + 2.0 ** -30) == 1 + u  # just above tie
    assert round_bf16(255.5) == 256.0                 # binade carry
    assert bf16_from_bits(bf16_bits(round_bf16(3.03125)))[()] == 3.03125


def test_bits_roundtrip():
    x = np.array([0.0, -0.0, 1.0, -2.5, 65504.0, 2.0 ** -24])
    assert np.array_equal(fp16_bits(x).view(np.float16).astype(np.float64), x)
    assert fp16_bits(np.array([-0.0]))[0] == 0x8000


def test_ulp_matches_numpy_spacing_fp16():
    from oracle.numerics import ulp
    x = np.array([1.0, 3.0, 32768.0, 2.0 ** -14, 2.0 ** -20, 1000.0, 0.1])
    ref = np.abs(np.spacing(x.astype(np.float16)).astype(np.float64))
    assert np.array_equal(ulp(x, "fp16"), ref)
    assert ulp(0.0, "fp16") == 2.0 ** -24


def test_ulp_bf16():
    from oracle.numerics import ulp
    assert ulp(1.0, "bf16") == 2.0 ** -7
    assert ulp(3.0, "bf16") == 2.0 ** -6
    assert ulp(-5.0, "bf16") == 2.0 ** -5
    # the ulp is the step between consecutive bf16 values (independent bit-level check)
    import struct
    for v in (1.0, 3.5, 1e-3, 300.0):
        b = struct.unpack("<I", struct.pack("<f", v))[0] >> 16
        nxt = struct.unpack("<f", struct.pack("<I", (b + 1) << 16))[0]
        cur = struct.unpack("<f", struct.pack("<I", b << 16))[0]
        assert ulp(cur, "bf16") == nxt - cur
