"""Pins for oracle/moe.py (grouped MoE GEMM) against a plain GEMM and special cases."""

import numpy as np

from oracle.gemm import gemm_f64
from oracle.moe import grouped_gemm_f64
from paper_2508_15601_b200 import synth


def _experts(E, N, K, g, seed):
    ds = [synth.awq_like(1, N, K, group=g, seed=seed + e) for e in range(E)]
    return [d["q"] for d in ds], np.stack([d["s"] for d in ds]), np.stack([d["z"] for d in ds])


def test_one_expert_is_plain_gemm():
    qs, s, z = _experts(1, 256, 256, 128, 1)
    A = synth.awq_like(5, 256, 256, seed=9)["A"]
    assert np.array_equal(grouped_gemm_f64(A, qs, s, z, 128, [5]), gemm_f64(A, qs[0], s[0], z[0], 128))


def test_block_diagonal_embedding_equals_grouped():
    """Grouped result == one plain GEMM with A' = block-diagonal rows over K' = E*K and W' = the
    experts' weights stacked along K (zeros add nothing: exact in fp64)."""
    E, N, K, g = 4, 128, 256, 64
    m = [3, 0, 5, 2]
    qs, s, z = _experts(E, N, K, g, 20)
    A = synth.awq_like(sum(m), N, K, seed=21)["A"].astype(np.float64)
    Ap = np.zeros((sum(m), E * K))
    r = 0
    for e, me in enumerate(m):
        Ap[r:r + me, e * K:(e + 1) * K] = A[r:r + me]
        r += me
    qp = np.concatenate(qs, axis=0)
    sp = np.concatenate(list(s), axis=0)
    zp = np.concatenate(list(z), axis=0)
    assert np.array_equal(grouped_gemm_f64(A, qs, s, z, g, m), gemm_f64(Ap, qp, sp, zp, g))


def test_experts_without_tokens_contribute_nothing():
    qs, s, z = _experts(3, 128, 128, 128, 30)
    A = synth.awq_like(4, 128, 128, seed=31)["A"]
    C = grouped_gemm_f64(A, qs, s, z, 128, [0, 4, 0])
    assert np.array_equal(C, gemm_f64(A, qs[1], s[1], z[1], 128))
