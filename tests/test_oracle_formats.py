"""Pins for oracle/formats.py: hand-worked words, format round trips, the bit-plane identity."""

import numpy as np

from oracle import formats as F
from oracle.gemm import gemm_f64
from paper_2508_15601_b200 import synth


def test_awq_hand_worked_word():
    """Columns 0..7 with codes 1..8: nibbles hold columns (0,2,4,6,1,3,5,7) -> 0x86427531."""
    codes = np.arange(1, 9, dtype=np.uint8)[None, :]
    w = F.awq_pack_cols(codes)
    assert w.view(np.uint32)[0, 0] == 0x86427531
    assert np.array_equal(F.awq_unpack_cols(np.array([[np.uint32(0x86427531).view(np.int32)]]), 8), codes)


def test_gptq_hand_worked_word_and_v1_offset():
    """Rows 0..7 of one column with codes 1..8 -> 0x87654321; stored zero 4 means zero 5 in v1."""
    q = np.arange(1, 9, dtype=np.uint8)[:, None].repeat(8, axis=1)
    qw, qz = F.gptq_pack(q, np.full((1, 8), 5), zero_offset=1)
    assert np.all(qw.view(np.uint32) == 0x87654321)
    assert np.all(qz.view(np.uint32) == 0x44444444)
    q2, z2 = F.gptq_unpack(qw, qz, 8, zero_offset=1)
    assert np.array_equal(q2, q) and np.all(z2 == 5)


def test_round_trips_random():
    d = synth.uniform(1, 256, 512, group=128, seed=11)
    q, z = d["q"], d["z"].astype(np.int64)
    qw = F.awq_pack_cols(q)
    qz = F.awq_pack_cols(z.astype(np.uint8))
    q2, z2 = F.awq_unpack(qw, qz, 256)
    assert np.array_equal(q2, q) and np.array_equal(z2, d["z"])
    for off in (0, 1):
        zz = np.clip(z, off, 15)
        gw, gz = F.gptq_pack(q, zz, zero_offset=off)
        q3, z3 = F.gptq_unpack(gw, gz, 256, zero_offset=off)
        assert np.array_equal(q3, q) and np.array_equal(z3.astype(np.int64), zz)


def test_bitplane_hand_worked():
    """q8 = 0xB7 = 183, z8 = 0x2C = 44: 16 (11 - 2) + (7 - 12) = 139 = 183 - 44."""
    q4, s4, z4 = F.w8_bitplanes(np.array([[0xB7]], dtype=np.uint8), np.array([[0.5]], dtype=np.float16),
                                np.array([[0x2C]]))
    assert q4[:, 0].tolist() == [11, 7] and z4[:, 0].tolist() == [2, 12] and s4[:, 0].tolist() == [8.0, 0.5]
    assert (q4[0, 0] - z4[0, 0]) * s4[0, 0] + (q4[1, 0] - z4[1, 0]) * s4[1, 0] == (183 - 44) * 0.5


def test_bitplane_gemm_identity():
    """The W8A16 product equals the W4A16 product over 2K rows with [A | A] (fp64, to rounding)."""
    rng = np.random.default_rng(5)
    K, N, g, M = 256, 128, 64, 3
    q8 = rng.integers(0, 256, (K, N), dtype=np.uint8)
    z8 = rng.integers(0, 256, (K // g, N))
    s = rng.uniform(1e-3, 1e-2, (K // g, N)).astype(np.float16)
    A = rng.normal(size=(M, K))
    q4, s4, z4 = F.w8_bitplanes(q8, s, z8)
    ref = F.w8a16_gemm_f64(A, q8, s, z8, g)
    got = gemm_f64(np.concatenate([A, A], axis=1), q4, s4, z4, g)
    assert np.allclose(got, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
