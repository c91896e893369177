"""The paper's five §4 test problems:
pins of the generators' structure, of the oracle's constraint bounds against the
values the paper prints, and of the oracle's RQI against the paper's stated
behaviour on them.  CPU only."""
import math
import os

import numpy as np
import pytest

import tlsgen
from oracle import exact, rqi

GOLD = os.path.join(os.path.dirname(__file__), "golden", "paper_sec4_bounds.txt")


def _printed_bounds():
    out = {}
    with open(GOLD) as fh:
        for line in fh:
            if line.startswith("#") or not line.strip():
                continue
            f = line.split()
            out[f[0]] = (float(f[1]), float(f[2]))
    return out


def test_vanhuffel_matches_printed_system():
    """PAPER.md:596-613 at n = 4 (SPEC.md example): rows (3,-1), (-1,3), (-1,-1),
    (-1,-1); b = (-1,-1,3,-1).  A^T A = n^2 I - n J in closed form, so its eigenvalues
    are n^2 (n-3 times) and 2n."""
    P = tlsgen.paper_problem("vanhuffel", n=4, eps=0.0)
    assert np.array_equal(P.A, np.array([[3, -1], [-1, 3], [-1, -1], [-1, -1]], float))
    assert np.array_equal(P.b, np.array([-1, -1, 3, -1], float))
    n = 100
    P = tlsgen.paper_problem("vanhuffel", n=n, eps=0.0)
    G = P.A.T @ P.A
    assert np.array_equal(G, n * n * np.eye(n - 2) - n * np.ones((n - 2, n - 2)))
    ev = np.linalg.eigvalsh(G)
    assert ev[0] == pytest.approx(2 * n) and ev[-1] == pytest.approx(n * n)


def test_delta_and_bjorck_singular_values():
    """delta matrix: singular values {delta, delta, 1, 1} unperturbed.
    Bjorck: sigma_i(A) = 2^{-(i-1)} and b = A x consistent."""
    P = tlsgen.paper_problem("delta", eps=0.0)
    assert np.allclose(np.sort(np.linalg.svd(P.A, compute_uv=False)), [1e-2, 1e-2, 1, 1], rtol=1e-15)
    P = tlsgen.paper_problem("bjorck", eps=0.0)
    s = np.linalg.svd(P.A, compute_uv=False)
    assert np.allclose(s, 2.0 ** -np.arange(15), rtol=1e-12)
    ex = exact.tls_svd(P.A, P.b)
    assert ex.sigma < 1e-14 * s[0]
    assert np.allclose(ex.x, 1.0 / np.arange(1, 16), rtol=1e-9)


def test_toeplitz_band():
    """column j of Tbar holds t_1..t_{2w+1} on rows j..j+2w; each
    column sums to the truncated Gaussian mass sum_i t_i."""
    P = tlsgen.paper_problem("toeplitz", eps=0.0)
    w, a = 2, 1.25
    t = np.array([math.exp(-((w - i + 1) ** 2) / (2 * a * a)) / math.sqrt(2 * math.pi * a * a)
                  for i in range(1, 2 * w + 2)])
    assert P.A.shape == (100, 96)
    assert np.allclose(P.A.sum(axis=0), t.sum(), rtol=1e-14)
    assert np.array_equal(P.A[3:8, 3], t)
    assert np.count_nonzero(P.A) == 96 * (2 * w + 1)


@pytest.mark.parametrize("name,which,factor", [("random", 0, 3), ("random", 1, 4), ("delta", 0, 3),
                                               ("delta", 1, 3), ("bjorck", 0, 3), ("vanhuffel", 0, 3),
                                               ("vanhuffel", 1, 3)])
def test_constraint_bounds_match_printed(name, which, factor):
    """exact.constraints (constr1/constr2) on our instances
    lands within a small factor of the bound the paper prints for its own instance of
    the same distribution (tests/golden/paper_sec4_bounds.txt), for every seed 1..6.
    Not pinned: bjorck constr2 (the gap 1 - sigma^2/sigma'^2 varies 100x over seeds)
    and toeplitz (the printed '<~ 1' is not reproduced by any reading of the garbled
    definition: the band's symbol has zeros on the unit circle, kappa ~ 400; R21)."""
    printed = _printed_bounds()[name][which]
    for seed in range(1, 7):
        P = tlsgen.paper_problem(name, seed=seed)
        c = exact.constraints(P.A, exact.tls_svd(P.A, P.b))
        got = c["constr1" if which == 0 else "constr2"]
        assert printed / factor <= got <= printed * factor, (seed, got)


@pytest.mark.parametrize("name", ["random", "vanhuffel", "toeplitz"])
def test_mp_delay_and_same_limiting_accuracy(name):
    """the mixed precision variant may take more RQI
    steps than the uniform one (here: the u_f = fp64 control), and both reach a
    similar limiting accuracy.  Checked against the SVD of [A, b]."""
    P = tlsgen.paper_problem(name)
    ex = exact.tls_svd(P.A, P.b)
    _, ref = rqi.solve(P.A, P.b, "fp64")
    for fmt in ("fp16", "bf16"):
        _, r = rqi.solve(P.A, P.b, fmt)
        assert r.status == rqi.OK
        assert r.rqi_iters >= ref.rqi_iters or ref.status != rqi.OK
        assert np.linalg.norm(r.x - ex.x) / np.linalg.norm(ex.x) <= 1e-12
        assert abs(r.sigma - ex.sigma) / ex.sigma <= 1e-13
