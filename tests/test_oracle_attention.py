"""Pins for oracle/attention.py (low-bit-KV decode attention)."""

from fractions import Fraction

import numpy as np
import pytest

from oracle.attention import decode_attention_f64, dequant_kv
from paper_2508_15601_b200 import synth


def _one(Lmax=64, L=None, bits=8, B=1, Hq=4, Hkv=1, D=128, seed=1):
    return synth.kv_decode_problem(B, Hq, Hkv, D, Lmax, [L or Lmax] * B, bits, seed=seed)


def _run(p, **kw):
    return decode_attention_f64(p["Q"], p["kq"], p["ks"], p["kz"], p["vq"], p["vs"], p["vz"], p["seq_lens"], **kw)


def test_single_token_returns_its_value():
    p = _one(L=1)
    O = _run(p)
    V0 = dequant_kv(p["vq"][0, 0, 0], p["vs"][0, 0, 0], p["vz"][0, 0, 0])
    for h in range(4):
        assert np.array_equal(O[0, h], V0)


def test_identical_keys_and_zero_query_give_mean_value():
    p = _one(L=5)
    p["kq"][0, 0, :5] = p["kq"][0, 0, 0]
    p["ks"][0, 0, :5] = p["ks"][0, 0, 0]
    p["kz"][0, 0, :5] = p["kz"][0, 0, 0]
    V = dequant_kv(p["vq"][0, 0, :5], p["vs"][0, 0, :5], p["vz"][0, 0, :5])
    assert np.allclose(_run(p)[0, 0], V.mean(axis=0), rtol=0, atol=1e-13)
    p2 = _one(L=7, seed=2)
    p2["Q"][:] = 0.0
    V2 = dequant_kv(p2["vq"][0, 0, :7], p2["vs"][0, 0, :7], p2["vz"][0, 0, :7])
    assert np.allclose(_run(p2)[0, 2], V2.mean(axis=0), rtol=0, atol=1e-13)


def test_dominant_key_selects_its_value():
    p = _one(L=9, bits=8, seed=3)
    q = p["Q"][0, 1].astype(np.float64)
    # key 4 = large multiple of q's sign pattern: its score dominates all others by > 700 nats
    p["kq"][0, 0, 4] = np.where(q > 0, 255, 0)
    p["kz"][0, 0, 4] = 128
    p["ks"][0, 0, 4] = 1.0
    O = _run(p)
    V4 = dequant_kv(p["vq"][0, 0, 4], p["vs"][0, 0, 4], p["vz"][0, 0, 4])
    assert np.allclose(O[0, 1], V4, rtol=0, atol=1e-12)


def test_shift_invariance():
    """Adding the same vector c*q/|q|^2-direction offset to every key adds a constant to every
    score: O is unchanged.  Done exactly on the integer codes: raising every key's zero point by
    one shifts K[t] by -s_t, so use equal scales to make the shift a constant."""
    p = _one(L=16, bits=4, seed=4)
    p["ks"][0, 0, :] = np.float16(0.25)
    O1 = _run(p)
    p["kz"][0, 0, :] = p["kz"][0, 0, :] + 1   # K[t] -> K[t] - 0.25 for every t: S shifts by -0.25 sum(q)/sqrt(D)
    O2 = _run(p)
    assert np.allclose(O1, O2, rtol=0, atol=1e-12)


def test_exact_rational_dot_products_tiny():
    """Scores from exact rational dot products, softmax and P.V in float64 from them: matches."""
    p = _one(Lmax=64, L=6, bits=4, Hq=2, Hkv=1, D=16, seed=5)
    O = _run(p)
    K = dequant_kv(p["kq"][0, 0, :6], p["ks"][0, 0, :6], p["kz"][0, 0, :6])
    V = dequant_kv(p["vq"][0, 0, :6], p["vs"][0, 0, :6], p["vz"][0, 0, :6])
    for h in range(2):
        S = [float(sum(Fraction(float(a)) * Fraction(float(b)) for a, b in zip(p["Q"][0, h], K[t]))) / 4.0
             for t in range(6)]
        m = max(S)
        e = [np.exp(x - m) for x in S]
        tot = sum(e)
        ref = [sum(e[t] / tot * V[t, d] for t in range(6)) for d in range(16)]
        assert np.allclose(O[0, h], ref, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("bits", [4, 8])
def test_kv_quantisation_round_trip(bits):
    rng = np.random.default_rng(bits)
    X = rng.normal(size=(3, 5, 128)).astype(np.float32)
    q, s, z = synth.quantize_kv(X, bits)
    assert q.max() <= (1 << bits) - 1
    err = np.abs(dequant_kv(q, s, z) - X)
    assert np.all(err <= s.astype(np.float64)[..., None] / 2 + 1e-6)
