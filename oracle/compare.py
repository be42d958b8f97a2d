"""Parity metrics for the GEMM (test infrastructure; see oracle/__init__.py).

The north star fixes two criteria for GEMM output against the oracle:
  (a) relative Frobenius error  ||C_gpu - C_ref||_F / ||C_ref||_F <= 5e-3
  (b) per-element |C_gpu - C_ref| <= 1e-2 * sqrt(K/128) * max|A| * max|scale|

Reading R12, implemented here line for line:
  * B = 1e-2 * sqrt(K/128) * max|A| * S, where
      S = max|s|             for fp16 outputs (the literal wording), and
      S = max|s * (q - z)|   for bf16 outputs and fp32 partials: the largest dequantised
                             weight, taken element by element over the whole weight
                             (max_dequant_weight), NOT max|s| * max|q - z|.
  * bound = B + 0.5 * ulp_out(C_ref) for bf16/fp16 outputs; bound = B for fp32 partials.
    The half-ulp term is the one final rounding of C to the output dtype (reading R8):
    the correctly rounded exact result itself differs from C_ref by up to half an output
    ulp, independently of K, so a bound without it could reject the exact answer (e.g.
    C_ref = 1 + 2^-9 when B < 2^-9).  fp32 partials are not rounded by the kernel.
  * (a) is the primary gate; `ok` requires (a), (b) and finite outputs.
`check` also reports `max_ratio_strict` = max |err| / B (no half-ulp term), so every test
can state the ratio under the narrower reading as well.
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


def max_dequant_weight(q, scales, zeros, group, col_block=4096):
    """max over (k, n) of |s[k//g][n] * (q[k][n] - z[k//g][n])| in float64 (exact: a
    4-5 bit integer times an fp16 value)."""
    q = np.asarray(q)
    K, N = q.shape
    if q.size == 0:
        return 0.0
    s = np.asarray(scales, dtype=np.float64)
    z = np.asarray(zeros, dtype=np.float64)
    best = 0.0
    for c0 in range(0, N, col_block):
        cols = slice(c0, min(N, c0 + col_block))
        qc = (q[:, cols].astype(np.int64) & 0xF).astype(np.float64).reshape(K // group, group, -1)
        w = np.abs((qc - z[:, None, cols]) * s[:, None, cols])
        best = max(best, float(w.max()))
    return best


def elem_bound(A, scales, zeros, q, group, out_dtype):
    """B, the accumulated-error part of the per-element bound under reading R12."""
    A = np.asarray(A)
    K = np.asarray(q).shape[0]
    amax = float(np.max(np.abs(np.asarray(A, dtype=np.float64)))) if A.size else 0.0
    base = 1e-2 * np.sqrt(K / 128.0) * amax
    if out_dtype == "fp16":
        return base * float(np.max(np.abs(np.asarray(scales, dtype=np.float64))))
    return base * max_dequant_weight(q, scales, zeros, group)


def check(C, C_ref, A, q, scales, zeros, group, out_dtype):
    """Returns a dict: relfro, max_abs_err, bound (= B), max_ratio (B + half-ulp),
    max_ratio_strict (B alone), argmax (of max_ratio), ok."""
    C = np.asarray(C, dtype=np.float64)
    C_ref = np.asarray(C_ref, dtype=np.float64)
    err = np.abs(C - C_ref)
    B = elem_bound(A, scales, zeros, q, group, out_dtype)
    bound = B + (0.5 * ulp(C_ref, out_dtype) if out_dtype in ("bf16", "fp16") else 0.0)

    def _ratio(bd):
        bd = np.broadcast_to(np.asarray(bd, dtype=np.float64), err.shape)
        with np.errstate(divide="ignore", invalid="ignore"):
            return np.where(bd > 0, err / np.where(bd > 0, bd, 1.0), np.where(err > 0, np.inf, 0.0))

    ratio = _ratio(bound)
    idx = np.unravel_index(int(np.argmax(ratio)), ratio.shape) if ratio.size else ()
    max_ratio = float(ratio[idx]) if ratio.size else 0.0
    max_strict = float(_ratio(B).max()) if ratio.size else 0.0
    rf = relfro(C, C_ref)
    ok = bool(np.all(np.isfinite(C))) and rf <= RELFRO_TOL and max_ratio <= 1.0
    return dict(relfro=rf, max_abs_err=float(err.max()) if err.size else 0.0, bound=B,
                max_ratio=max_ratio, max_ratio_strict=max_strict,
                argmax=tuple(int(i) for i in idx), ok=ok)


def summary(r):
    """One-line description for assertion messages."""
    return (f"relfro={r['relfro']:.3e} max_ratio={r['max_ratio']:.3f} "
            f"max_ratio_strict={r['max_ratio_strict']:.3f} argmax={r['argmax']} ok={r['ok']}")
