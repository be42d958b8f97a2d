"""Software round-to-nearest-even (RNE) from float64 to bf16 and fp16.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Why the oracle needs its own rounding: the dequantised weight and the output C
are rounded to the activation dtype at designated points (DESIGN.md §4 readings
R6, R8; §3.1 step (iii) "dequantizing the INT4 values to FP16",
P:181; "nearest binary16 value, ties to even; overflow saturates to
signed infinity").  numpy has no bfloat16, so both formats are written here as
one generic rule:

    for finite x != 0 with |x| = m * 2**E, 0.5 <= m < 1 (frexp):
        e      = max(E - 1, emin)            # exponent of the binade (subnormals clamp)
        quantum = 2 ** (e - (p - 1))          # spacing of representable values there
        r      = rint(x / quantum) * quantum  # rint is round-half-to-even
        |r| > max_finite  ->  +-inf

with (p, emin, max_finite) = (8, -126, (2 - 2**-7) * 2**127) for bf16 and
(11, -14, 65504) for fp16.  x / quantum is exact in float64 because quantum is
a power of two and every input here lies well inside float64's range.

Pinned by tests/test_oracle_numerics.py: numpy's own float64->float16 cast (a
correctly-rounded library conversion) on random and tie-crafted values, an
independent integer bit-trick RNE for float32->bf16, torch's float32->bfloat16
cast, and the SPEC.md S:49-54 examples (2049 -> 2048, 65520 -> inf).
"""

import numpy as np

BF16 = dict(p=8, emin=-126, max_finite=(2.0 - 2.0 ** -7) * 2.0 ** 127)
FP16 = dict(p=11, emin=-14, max_finite=65504.0)


def _rne(x, p, emin, max_finite):
    x = np.asarray(x, dtype=np.float64)
    out = np.array(x, dtype=np.float64, copy=True)
    finite = np.isfinite(x) & (x != 0.0)
    xf = x[finite]
    _, E = np.frexp(xf)
    e = np.maximum(E - 1, emin)
    quantum = np.ldexp(1.0, e - (p - 1))
    r = np.rint(xf / quantum) * quantum
    r = np.where(np.abs(r) > max_finite, np.copysign(np.inf, xf), r)
    out[finite] = r
    return out


def round_bf16(x):
    """RNE float64 -> bf16, returned as float64 values (exactly representable in bf16)."""
    return _rne(x, **BF16)


def round_fp16(x):
    """RNE float64 -> fp16, returned as float64 values (exactly representable in fp16)."""
    return _rne(x, **FP16)


def ulp(x, dtype):
    """Spacing of `dtype` values at |x| (the binade's quantum; subnormal spacing below
    the smallest normal).  Used for the half-ulp output-rounding allowance (reading R12)."""
    fmt = BF16 if dtype == "bf16" else FP16
    x = np.abs(np.asarray(x, dtype=np.float64))
    _, E = np.frexp(x)  # frexp(0) gives E = 0, clamped to emin below (subnormal spacing)
    e = np.maximum(np.where(x > 0, E - 1, fmt["emin"]), fmt["emin"])
    return np.ldexp(1.0, e - (fmt["p"] - 1))


def round_to(x, dtype):
    """dtype in {'bf16', 'fp16'}."""
    if dtype == "bf16":
        return round_bf16(x)
    if dtype == "fp16":
        return round_fp16(x)
    raise ValueError(dtype)


def bf16_bits(x):
    """uint16 bit patterns of values already representable in bf16."""
    f = np.asarray(x, dtype=np.float64).astype(np.float32)
    return (f.view(np.uint32) >> 16).astype(np.uint16)


def fp16_bits(x):
    """uint16 bit patterns of values already representable in fp16."""
    return np.asarray(x, dtype=np.float64).astype(np.float16).view(np.uint16)


def bf16_from_bits(b):
    b = np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16
    return b.view(np.float32).astype(np.float64)


def fp16_from_bits(b):
    return np.asarray(b, dtype=np.uint16).view(np.float16).astype(np.float64)
