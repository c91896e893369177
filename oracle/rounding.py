"""Direct fp64 -> u_f rounding, round-to-nearest-even (oracle; test infrastructure).

PAPER.md Table 2 (l.435-447) lists the unit roundoffs of fp16 (4.88e-4),
fp32 (5.96e-8) and fp64 (1.11e-16); bf16 is absent from the paper and is read
as p = 8 significand bits with fp32's exponent range (reading R12).
The paper simulates low precision with `chop` (l.480); it does not state the
rounding mode, so round-to-nearest-even with gradual underflow and overflow to
+-inf is taken (reading R4).  Rounding is DIRECT from fp64 (no
intermediate fp32 step, which would double-round for bf16).

The rule, written out for a finite x != 0 with significand precision p and
minimum normal exponent emin, maximum exponent emax:
    e  = floor(log2 |x|)                 (exact, from frexp)
    q  = 2^(max(e, emin) - (p - 1))      (the spacing of the target format at x)
    y  = q * round_half_even(x / q)      (x / q is exact: q is a power of two)
    |y| > (2 - 2^(1-p)) * 2^emax  ->  y = +-inf
"""
from __future__ import annotations

import numpy as np

# name -> (p, emin, emax)
FORMATS = {
    "fp16": (11, -14, 15),
    "bf16": (8, -126, 127),
    "fp32": (24, -126, 127),
    "fp64": (53, -1022, 1023),
}


def unit_roundoff(fmt: str) -> float:
    """u = 2^-p (Table 2, l.442-444)."""
    p = FORMATS[fmt][0]
    return 2.0 ** (-p)


def max_finite(fmt: str) -> float:
    p, _, emax = FORMATS[fmt]
    return (2.0 - 2.0 ** (1 - p)) * 2.0 ** emax


def round_to(x, fmt: str) -> np.ndarray:
    """Round fp64 values to the nearest `fmt` value (ties to even); returns fp64."""
    x = np.asarray(x, dtype=np.float64)
    if fmt == "fp64":
        return x.copy()
    p, emin, emax = FORMATS[fmt]
    out = x.copy()
    fin = np.isfinite(x) & (x != 0.0)
    xf = x[fin]
    _, E = np.frexp(xf)             # xf = f * 2^E, 0.5 <= |f| < 1
    e = E.astype(np.int64) - 1      # floor(log2 |xf|)
    q = np.ldexp(1.0, np.maximum(e, emin) - (p - 1))
    y = np.rint(xf / q) * q         # np.rint rounds half to even
    y = np.where(np.abs(y) > max_finite(fmt), np.copysign(np.inf, xf), y)
    out[fin] = y
    return out
