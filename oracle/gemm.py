"""The W4A16 GEMM, oracle side: C = A . dequant(q, s, z) in float64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

What the method computes ("the result, plainly"): the online GEMM
of PAPER.md §3.4 feeds dequantised weights "alongside the FP16
activations to perform standard FP16 matrix multiplication" (§3.1 step (iv),
P:181), so the result is the plain definition

    C[m][n] = sum_{k<K} A[m][k] * (q[k][n] - z[k//g][n]) * s[k//g][n]

rounded once to the output dtype (north star: "fp32 accumulation", "bf16 C";
SPEC.md S:374-377).  The oracle evaluates the sum in float64 on the exact fp64
dequantised weights (dequant_f64), using numpy's fp64 matmul as the one library
primitive, in column blocks only to bound memory (70B shapes would need 3.8 GB of
fp64 weights otherwise).  No output rounding is applied here; the comparison
metrics (oracle/compare.py) and the closed-form tests round with
oracle/numerics.py where a bit-exact claim is made.

Pinned by tests/test_oracle_gemm.py: exact rational brute force (Python
fractions, triple loop) on the tiny config, zero weights -> 0,
one-hot activation rows -> the dequantised weight row, all-ones A with
power-of-two scales -> integer column sums times s, and exact doubling under A*2.
"""

import numpy as np

from .quant import dequant_f64


def gemm_f64(A, q, scales, zeros, group, rows=None, col_block=4096):
    """C (float64 [len(rows) or M][N]) = A[rows] . dequant_f64(q, s, z).

    A: float array [M][K] holding the activation values exactly (bf16/fp16 values).
    q: uint8 [K][N]; scales, zeros: [K/group][N]."""
    A = np.asarray(A, dtype=np.float64)
    if rows is not None:
        A = A[np.asarray(rows)]
    K, N = np.asarray(q).shape
    if A.shape[1] != K:
        raise ValueError("A.shape[1] must equal K")
    C = np.empty((A.shape[0], N), dtype=np.float64)
    for c0 in range(0, N, col_block):
        cols = slice(c0, min(N, c0 + col_block))
        W = dequant_f64(q, scales, zeros, group, cols=cols)
        C[:, cols] = A @ W
    return C
