"""Pins for oracle/gemm.py against exact rational brute force, closed forms and invariants."""

from fractions import Fraction

import numpy as np
import pytest

from oracle.gemm import gemm_f64
from oracle.quant import dequant_f64
from oracle import compare
from paper_2508_15601_b200 import synth


def _brute_fraction(A, q, s, z, group, rows, cols):
    """Pure-Python exact rational triple loop over the paper's definition
    C[m][n] = sum_k A[m][k] (q[k][n] - z[k//g][n]) s[k//g][n]."""
    K = q.shape[0]
    out = {}
    for m in rows:
        for n in cols:
            acc = Fraction(0)
            for k in range(K):
                w = (Fraction(int(q[k, n]) & 0xF) - Fraction(float(z[k // group, n]))) * Fraction(float(s[k // group, n]))
                acc += Fraction(float(A[m, k])) * w
            out[(m, n)] = acc
    return out


def test_tiny_config_vs_exact_rationals():
    """CFG#0 (M=4, N=256, K=256, group=128): fp64 oracle within 1e-12 relative of exact."""
    d = synth.awq_like(4, 256, 256, group=128, seed=1000)
    C = gemm_f64(d["A"], d["q"], d["s"], d["z"], 128)
    ex = _brute_fraction(d["A"], d["q"], d["s"], d["z"], 128, range(4), range(0, 256, 5))
    scale = max(abs(float(v)) for v in ex.values())
    for (m, n), v in ex.items():
        assert abs(C[m, n] - float(v)) <= 1e-12 * scale


def test_uniform_vs_exact_rationals_group64():
    d = synth.uniform(3, 128, 192, group=64, seed=7)
    C = gemm_f64(d["A"], d["q"], d["s"], d["z"], 64)
    ex = _brute_fraction(d["A"], d["q"], d["s"], d["z"], 64, range(3), range(0, 128, 9))
    scale = max(abs(float(v)) for v in ex.values())
    for (m, n), v in ex.items():
        assert abs(C[m, n] - float(v)) <= 1e-12 * scale


def test_zero_weights():
    """q == z everywhere -> C == 0."""
    rng = np.random.default_rng(1)
    K, N, g = 256, 256, 128
    z = rng.integers(0, 16, size=(K // g, N)).astype(np.float16)
    q = np.repeat(z.astype(np.uint8), g, axis=0)
    s = rng.uniform(0.001, 0.1, size=(K // g, N)).astype(np.float16)
    A = rng.normal(size=(5, K))
    assert np.all(gemm_f64(A, q, s, z, g) == 0.0)


def test_onehot_rows_give_dequant_rows():
    d = synth.uniform(1, 256, 256, group=128, seed=9)
    A = np.zeros((6, 256))
    ks = [0, 1, 63, 64, 128, 255]
    for m, k in enumerate(ks):
        A[m, k] = 1.0
    C = gemm_f64(A, d["q"], d["s"], d["z"], 128)
    W = dequant_f64(d["q"], d["s"], d["z"], 128)
    for m, k in enumerate(ks):
        assert np.array_equal(C[m], W[k])


def test_ones_activation_power_of_two_scales():
    """A = 1, s = 2^-j: C[n] = 2^-j * sum_k (q - z), an exact integer sum."""
    rng = np.random.default_rng(12)
    K, N, g = 512, 128, 128
    q = rng.integers(0, 16, size=(K, N), dtype=np.uint8)
    z = rng.integers(0, 16, size=(K // g, N)).astype(np.float16)
    s = np.full((K // g, N), 2.0 ** -5, dtype=np.float16)
    C = gemm_f64(np.ones((2, K)), q, s, z, g)
    expect = 2.0 ** -5 * (q.astype(np.int64) - np.repeat(z.astype(np.int64), g, axis=0)).sum(axis=0)
    assert np.array_equal(C[0], expect) and np.array_equal(C[1], expect)


def test_doubling_is_exact():
    d = synth.awq_like(4, 128, 256, seed=3)
    C1 = gemm_f64(d["A"], d["q"], d["s"], d["z"], 128)
    C2 = gemm_f64(2.0 * d["A"].astype(np.float64), d["q"], d["s"], d["z"], 128)
    assert np.array_equal(C2, 2.0 * C1)


def test_rows_and_column_blocks_consistent():
    d = synth.awq_like(7, 384, 256, seed=4)
    C = gemm_f64(d["A"], d["q"], d["s"], d["z"], 128)
    Cb = gemm_f64(d["A"], d["q"], d["s"], d["z"], 128, col_block=128)
    Cr = gemm_f64(d["A"], d["q"], d["s"], d["z"], 128, rows=[6, 0, 3])
    np.testing.assert_allclose(Cb, C, rtol=1e-15, atol=0)
    np.testing.assert_allclose(Cr, C[[6, 0, 3]], rtol=1e-15, atol=0)


def test_compare_metrics():
    C = np.array([[1.0, 2.0], [3.0, 4.0]])
    assert compare.relfro(C, C) == 0.0
    assert compare.relfro(C * (1 + 1e-3), C) == pytest.approx(1e-3)
    q = np.zeros((128, 2), dtype=np.uint8)
    z = np.full((1, 2), 15, dtype=np.float16)
    s = np.full((1, 2), 0.5, dtype=np.float16)
    A = np.ones((2, 128))
    b_bf = compare.elem_bound(A, s, z, q, 128, "bf16")
    b_h = compare.elem_bound(A, s, z, q, 128, "fp16")
    assert b_h == pytest.approx(1e-2 * 0.5) and b_bf == pytest.approx(15 * 1e-2 * 0.5)
    r = compare.check(C * (1 + 1e-3), C, A, q, s, z, 128, "fp16")
    assert r["relfro"] == pytest.approx(1e-3) and r["argmax"] == (1, 1)


def test_compare_bound_is_max_dequant_weight_not_product_of_maxima():
    """Reading R12: S = max|s*(q-z)| element by element.  Here the largest scale sits in a
    group whose codes equal the zero (dequantised weight 0), and the largest |q-z| sits in a
    group with a small scale, so max|s|*max|q-z| = 2*15 = 30 while max|s*(q-z)| = 0.25*15."""
    K, N, g = 256, 128, 128
    q = np.zeros((K, N), dtype=np.uint8)
    z = np.zeros((K // g, N), dtype=np.float16)
    s = np.full((K // g, N), 0.25, dtype=np.float16)
    s[0, :] = 2.0                      # group 0: big scale, q == z -> weight 0
    q[g:, :] = 15                      # group 1: |q - z| = 15 at scale 0.25
    assert compare.max_dequant_weight(q, s, z, g) == 0.25 * 15
    A = np.ones((1, K))
    B = compare.elem_bound(A, s, z, q, g, "bf16")
    assert B == pytest.approx(1e-2 * np.sqrt(2.0) * 0.25 * 15)
    assert B < 1e-2 * np.sqrt(2.0) * 2.0 * 15 / 4          # the looser product reading is 8x larger
    # an error between the two readings is rejected under R12
    C_ref = np.zeros((1, N))
    C_ref[0, :] = 15 * 0.25 * g
    C = C_ref + 2.0 * B
    r = compare.check(C, C_ref, A, q, s, z, g, "fp32")
    assert not r["ok"] and r["max_ratio"] == pytest.approx(2.0) and r["max_ratio_strict"] == pytest.approx(2.0)
    # fp16 reads the literal max|s|
    assert compare.elem_bound(A, s, z, q, g, "fp16") == pytest.approx(1e-2 * np.sqrt(2.0) * 2.0)


def test_max_dequant_weight_column_blocks():
    d = synth.uniform(1, 384, 256, group=64, seed=5)
    full = float(np.max(np.abs(dequant_f64(d["q"], d["s"], d["z"], 64))))
    assert compare.max_dequant_weight(d["q"], d["s"], d["z"], 64, col_block=128) == full


def test_compare_half_ulp_allowance():
    """An output that is exactly the RNE of the reference passes even when the accumulated
    bound B is tiny (reading R12: one final output rounding is allowed half an ulp)."""
    from oracle.numerics import round_bf16
    rng = np.random.default_rng(0)
    C_ref = rng.normal(0, 3, size=(4, 128))
    q = np.zeros((128, 128), dtype=np.uint8)
    z = np.zeros((1, 128), dtype=np.float16)
    s = np.full((1, 128), 1e-4, dtype=np.float16)
    A = np.full((4, 128), 1e-3)
    r = compare.check(round_bf16(C_ref), C_ref, A, q, s, z, 128, "bf16")
    assert r["max_ratio"] <= 1.0
    assert r["max_ratio_strict"] > 1.0   # B alone (q == z: S = 0) would reject the exact answer
    # an error of one full ulp fails
    from oracle.numerics import ulp
    r = compare.check(C_ref + ulp(C_ref, "bf16"), C_ref, A, q, s, z, 128, "bf16")
    assert r["max_ratio"] > 1.0
