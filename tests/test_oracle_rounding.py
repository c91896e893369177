"""Pins for oracle/rounding.py (u_f rounding; Table 2 l.435-447).

Independent references: numpy's IEEE fp64->fp16 and fp64->fp32 conversions
(direct, round-to-nearest-even), the classic integer RNE on fp32 bit patterns
for bf16 of fp32-representable inputs, and exact rational arithmetic."""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle.rounding import round_to, unit_roundoff, max_finite, FORMATS

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _samples(rng, n=200000):
    # spread over many binades incl. fp16/bf16 subnormal, normal and overflow ranges
    e = rng.uniform(-160, 140, n)
    x = rng.choice([-1.0, 1.0], n) * np.exp2(e) * rng.uniform(1, 2, n)
    return x


def _ties(fmt, rng, n=5000):
    """Exact midpoints between consecutive values of the format (fp64-exact)."""
    p, emin, emax = FORMATS[fmt]
    e = rng.integers(emin - p + 1, emax, n)
    ee = np.maximum(e, emin)
    q = np.ldexp(1.0, ee - (p - 1))
    k = rng.integers(2 ** (p - 1), 2 ** p, n).astype(np.float64)
    k = np.where(e < emin, rng.integers(0, 2 ** (p - 1), n).astype(np.float64), k)
    return (k + 0.5) * q


@pytest.mark.parametrize("fmt,npdt", [("fp16", np.float16), ("fp32", np.float32)])
def test_bitexact_vs_ieee_cast(fmt, npdt):
    rng = np.random.default_rng(0)
    x = np.concatenate([_samples(rng), _ties(fmt, rng), -_ties(fmt, rng),
                        [0.0, -0.0, max_finite(fmt), 65519.99, 65520.0, 1e300, -1e300]])
    with np.errstate(over="ignore"):
        ref = x.astype(npdt).astype(np.float64)
    got = round_to(x, fmt)
    same = (got == ref) | (np.isnan(got) & np.isnan(ref))
    assert same.all(), x[~same][:5]
    # signed zeros preserved
    assert np.array_equal(np.signbit(got[ref == 0]), np.signbit(ref[ref == 0]))


def _bf16_from_f32_bits(x32: np.ndarray) -> np.ndarray:
    """Textbook RNE of fp32 bit patterns to the top 16 bits (valid for finite
    inputs that are exactly fp32; no double rounding because the input IS fp32)."""
    u = x32.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def test_bf16_vs_f32_bit_rne():
    rng = np.random.default_rng(1)
    with np.errstate(over="ignore"):
        x = _samples(rng).astype(np.float32)
    x = x[np.isfinite(x) & (np.abs(x) < 3e38)]
    ties = _ties("bf16", rng).astype(np.float32)
    x = np.concatenate([x, ties, -ties])
    ref = _bf16_from_f32_bits(x)
    got = round_to(x.astype(np.float64), "bf16")
    ok = (got == ref) | (np.isinf(got) & np.isinf(ref))
    assert ok.all(), x[~ok][:5]


def test_bf16_no_double_rounding_exact_rational():
    """fp64 values just above a bf16 midpoint must round UP, although rounding
    through fp32 first would land on the midpoint and then tie to even."""
    rng = np.random.default_rng(2)
    for _ in range(300):
        e = int(rng.integers(-120, 120))
        k = int(rng.integers(128, 256)) & ~1        # even significand -> tie goes down
        mid = (k + 0.5) * 2.0 ** (e - 7)
        above = mid * (1 + 2.0 ** -40)              # not fp32-representable, > mid
        below = mid * (1 - 2.0 ** -40)
        got_a = round_to(np.array([above]), "bf16")[0]
        got_b = round_to(np.array([below]), "bf16")[0]
        # exact nearest bf16 by rational comparison against the two neighbours
        lo, hi = k * 2.0 ** (e - 7), (k + 1) * 2.0 ** (e - 7)
        for v, got in ((above, got_a), (below, got_b)):
            dv = Fraction(v)
            nearest = lo if abs(dv - Fraction(lo)) < abs(dv - Fraction(hi)) else hi
            assert got == nearest
        # and the double-rounding path would be wrong for `above`
        via32 = _bf16_from_f32_bits(np.array([above], dtype=np.float32))[0]
        assert via32 == lo and got_a == hi


def test_table2_unit_roundoffs():
    """PAPER.md Table 2: printed values to the printed digits, and the measured
    worst relative rounding error is <= u and reaches ~u."""
    with open(os.path.join(GOLD, "table2_unit_roundoff.txt")) as fh:
        rows = [ln.split() for ln in fh if ln.strip() and not ln.startswith("#")]
    rng = np.random.default_rng(3)
    x = rng.uniform(1, 2, 100000) * np.exp2(rng.integers(-10, 10, 100000))
    for fmt, printed in rows:
        u = unit_roundoff(fmt)
        assert float(f"{u:.2e}") == float(printed)
        if fmt != "fp64":
            rel = np.max(np.abs(round_to(x, fmt) - x) / np.abs(x))
            assert rel <= u and rel > 0.99 * u
    assert unit_roundoff("bf16") == 2.0 ** -8       # reading R12 (not in the paper)


def test_invariants_idempotent_monotone():
    rng = np.random.default_rng(4)
    x = np.sort(_samples(rng, 50000))
    for fmt in ("fp16", "bf16", "fp32"):
        with np.errstate(invalid="ignore"):
            y = round_to(x, fmt)
            assert np.array_equal(round_to(y, fmt), y, equal_nan=True)
            fy = y[np.isfinite(y)]
            assert np.all(np.diff(fy) >= 0)


def test_overflow_and_subnormal_edges():
    assert round_to(np.array([65504.0]), "fp16")[0] == 65504.0
    assert math.isinf(round_to(np.array([65520.0]), "fp16")[0])        # tie -> even -> 2^16
    assert round_to(np.array([65519.0]), "fp16")[0] == 65504.0
    assert round_to(np.array([2.0 ** -24]), "fp16")[0] == 2.0 ** -24     # smallest subnormal
    assert round_to(np.array([2.0 ** -25]), "fp16")[0] == 0.0            # tie -> even 0
    assert round_to(np.array([2.0 ** -25 * 1.0000001]), "fp16")[0] == 2.0 ** -24
    assert round_to(np.array([2.0 ** -133]), "bf16")[0] == 2.0 ** -133   # bf16 min subnormal
