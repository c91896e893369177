"""Pins of the dense Gram accumulation bound (oracle.rqi.gram_accumulation_bound, reading R11)
against independent emulations of the accumulation family R11 names: K_t-row chunks summed in
fp32 with a TRUNCATING (round-toward-zero) or round-to-nearest adder, `super_chunks` chunk sums
added in fp32 (RNE), then fp64 -- compared with the exact sum of the exact products
(math.fsum).  The GPU's Gram (tcgen05, K_t = 64 rows per TMEM chunk, 64 chunk sums per fp64
flush) is tested against this bound in tests/test_gpu_parity.py."""
import math

import numpy as np
import pytest

from oracle import rqi
from oracle.rounding import round_to


def _rnd32(x, mode):
    """fp64 -> fp32 with round-to-nearest-even ('rne') or round-toward-zero ('rtz')."""
    r = x.astype(np.float32)
    if mode == "rtz":
        over = np.abs(r.astype(np.float64)) > np.abs(x)
        r = np.where(over, np.nextafter(r, np.float32(0)), r)
    return r


def _emulate(Ah, K_t, sup, mode):
    """Sequential emulation: rows added one at a time into an fp32 chunk accumulator with the
    given rounding; chunk sums added in fp32 RNE, `sup` per fp64 flush; flushes in fp64."""
    m, n = Ah.shape
    G = np.zeros((n, n))
    s2 = np.zeros((n, n), dtype=np.float32)
    npend = 0
    for c0 in range(0, m, K_t):
        s1 = np.zeros((n, n), dtype=np.float32)
        for i in range(c0, min(m, c0 + K_t)):
            p = np.outer(Ah[i], Ah[i])                     # exact (u_f products fit in fp64)
            s1 = _rnd32(s1.astype(np.float64) + p, mode)
        s2 = _rnd32(s2.astype(np.float64) + s1.astype(np.float64), "rne")
        npend += 1
        if npend == sup:
            G += s2.astype(np.float64)
            s2[:] = 0
            npend = 0
    if npend:
        G += s2.astype(np.float64)
    return G


def _exact(Ah):
    n = Ah.shape[1]
    return np.array([[math.fsum(Ah[:, a] * Ah[:, b]) for b in range(n)] for a in range(n)])


def _data(m, n, positive, fmt, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, n)) * np.logspace(0, -2, n)[None, :]
    if positive:
        A = np.abs(A)
    d, _ = rqi.column_scaling(A)
    return A, d, round_to(A / d, fmt)


@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
@pytest.mark.parametrize("positive", [False, True])
@pytest.mark.parametrize("K_t,sup,m", [(64, 64, 5000), (16, 8, 3001), (64, 4, 2600)])
def test_bound_covers_truncating_two_level_sum(fmt, positive, K_t, sup, m):
    A, d, Ah = _data(m, 6, positive, fmt, 1 + K_t + m)
    ex = _exact(Ah)
    B = rqi.gram_accumulation_bound(A, d, fmt, K_t, sup, truncating=True, nsplit=1)
    err = np.abs(_emulate(Ah, K_t, sup, "rtz") - ex)
    assert np.all(err <= B)
    Bn = rqi.gram_accumulation_bound(A, d, fmt, K_t, sup, truncating=False, nsplit=1)
    assert np.all(np.abs(_emulate(Ah, K_t, sup, "rne") - ex) <= Bn)
    if positive:
        # not vacuous: a truncating adder on positive data loses a share of an ulp per add
        # (less for bf16, whose 16-bit products often fit the fp32 partial sum exactly), a
        # fixed fraction of the bound (a bound missing its K_t factor would fail above)
        assert np.max(err / B) >= 0.02


def test_oracle_gram_within_the_one_level_bound():
    """The oracle's gram_uf (fp32 BLAS per K_t chunk, fp64 across chunks) is a member of the
    round-to-nearest, super_chunks = 1 family: within that bound of the exact sum, and the
    one-level bound equals gram_exact_bound's closed form up to its last-order terms."""
    A, d, Ah = _data(4099, 8, False, "fp16", 3)
    ex = _exact(Ah)
    G = rqi.gram_uf(A, d, "fp16", 64)
    B1 = rqi.gram_accumulation_bound(A, d, "fp16", 64, 1, truncating=False, nsplit=1)
    assert np.all(np.abs(G - ex) <= B1)
    Bx = rqi.gram_exact_bound(A, d, "fp16", 64)
    assert np.allclose(B1, Bx, rtol=0.05)
