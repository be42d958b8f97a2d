"""Grouped (mixture-of-experts) W4A16 GEMM, oracle side.  TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py).

The paper evaluates MoE models (§5); SURVEY §8(f) NEXT-3 asks for their expert
GEMMs in one launch.  What is computed is the plain definition applied per expert: the rows of A
are grouped by expert (expert 0's m_0 tokens first, then expert 1's, ...) and

    C[r] = sum_k A[r][k] * (q_e[k][n] - z_e[k//g][n]) * s_e[k//g][n]     for r in expert e's rows,

i.e. gemm_f64 of each expert's row block with that expert's weight (oracle/gemm.py).

Pinned by tests/test_oracle_moe.py: one expert reduces to gemm_f64; the grouped result equals ONE
plain GEMM on the block-diagonal embedding (A' = rows of expert e placed in column block e of an
[M][E*K] matrix of zeros, W' = the experts' weights stacked along K), exactly in fp64; experts
without tokens contribute nothing.
"""

import numpy as np

from .gemm import gemm_f64


def grouped_gemm_f64(A, qs, scales, zeros, group, m_per_expert):
    """A [sum m_e][K]; qs[e] uint8 [K][N]; scales/zeros [E][K/g][N] -> C float64 [sum m_e][N]."""
    A = np.asarray(A, dtype=np.float64)
    N = np.asarray(qs[0]).shape[1]
    C = np.zeros((A.shape[0], N), dtype=np.float64)
    r0 = 0
    for e, m in enumerate(m_per_expert):
        if m:
            C[r0:r0 + m] = gemm_f64(A[r0:r0 + m], qs[e], scales[e], zeros[e], group)
        r0 += m
    return C
