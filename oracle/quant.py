"""Group dequantisation (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The method's dequantisation (§3.1 step (iii): "dequantizing the
INT4 values to FP16 format through bit manipulation operations, and applying the
quantization scales"; §3.4: "dequantized into FP16 format through the
Integer-to-Float (I2F) procedure") with the group structure and zero points of
the north star ("per-group fp16 scales and zero points, group 128";
"dequant(q)=(q-zero)*scale") and SPEC.md S:119 "v = fp16_round((code - zp) x
scale)".  Readings: R1 asymmetric with zeros, R2 groups of
`group` consecutive k per column n with s, z stored [K/group][N], R3 codes are
unsigned 0..15 after masking with 0xF, R4 zeros are fp16 holding integers.

Two functions:

* dequant_f64 -- the plain definition W[k][n] = (q[k][n] - z[k//g][n]) * s[k//g][n]
  evaluated exactly in float64 (a 5-bit integer times an 11-bit fp16 fits in 53
  bits).  This is what the GEMM oracle multiplies by.
  Pinned by tests/test_oracle_quant.py: SPEC S:122-123 worked examples (code 12,
  s 0.5, zp 4 -> 4.0; code == zp -> 0), and exact rational evaluation.

* dequant_rounded -- the rounding sequence the CUDA kernel DECLARES for its
  operand (DESIGN.md §4 reading R6), used only for the bit-exact test of
  tm_dequant_w4:
      bf16:  x  = 128 + q              (exact: the 0x4300 magic-number bf16)
             zb = RNE_bf16(128 + z)
             t  = RNE_bf16(x - zb)     (exact for integer z)
             out = RNE_bf16(t * RNE_bf16(s))
      fp16:  x  = 1024 + q             (exact: the 0x6400 magic-number fp16)
             zh = RNE_fp16(1024 + z)
             t  = RNE_fp16(x - zh)     (exact for integer z)
             out = RNE_fp16(t * s)
  Each operation is evaluated exactly in float64 and rounded once, which is the
  IEEE semantics of sub.rn / mul.rn.  For integer z this equals
  RNE(RNE_bf16(s) * (q - z)) (bf16) and SPEC S:119's RNE_fp16((q - z) * s) (fp16).
  Pinned by: the closed forms just stated, the worked example s = 1.005859375,
  q - z = 3 -> bf16 3.03125 / fp16 3.017578125 computed by hand in DESIGN.md §4.
"""

import numpy as np

from .numerics import round_bf16, round_fp16


def _expand_groups(a, K, group):
    """[K/group][N] -> [K][N] by repeating each group row `group` times."""
    a = np.asarray(a, dtype=np.float64)
    if a.shape[0] * group != K:
        raise ValueError("scales/zeros rows must equal K / group")
    return np.repeat(a, group, axis=0)


def dequant_f64(q, scales, zeros, group, cols=None):
    """Exact W[k][n] = (q - z) * s in float64.  `cols` optionally selects a column slice."""
    q = np.asarray(q)
    if cols is not None:
        q, scales, zeros = q[:, cols], np.asarray(scales)[:, cols], np.asarray(zeros)[:, cols]
    K = q.shape[0]
    qf = (q.astype(np.int64) & 0xF).astype(np.float64)
    s = _expand_groups(scales, K, group)
    z = _expand_groups(zeros, K, group)
    return (qf - z) * s


def dequant_rounded(q, scales, zeros, group, dtype):
    """The kernel's declared operand rounding sequence (see module docstring)."""
    q = np.asarray(q)
    K = q.shape[0]
    qf = (q.astype(np.int64) & 0xF).astype(np.float64)
    s = _expand_groups(scales, K, group)
    z = _expand_groups(zeros, K, group)
    if dtype == "bf16":
        x = 128.0 + qf
        zb = round_bf16(128.0 + z)
        t = round_bf16(x - zb)
        return round_bf16(t * round_bf16(s))
    if dtype == "fp16":
        x = 1024.0 + qf
        zh = round_fp16(1024.0 + z)
        t = round_fp16(x - zh)
        return round_fp16(t * s)
    raise ValueError(dtype)
