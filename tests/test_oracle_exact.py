"""Pins for oracle/exact.py (the definitional TLS result, §1 l.58-63)."""
import math
import os

import numpy as np
import pytest

import tlsgen
from oracle import exact

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _delta_matrix(delta):
    rows = []
    with open(os.path.join(GOLD, "delta_matrix.txt")) as fh:
        for ln in fh:
            if ln.strip() and not ln.startswith("#"):
                rows.append([delta if t == "d" else float(t) for t in ln.split()])
    return np.array(rows)


def test_2x2_closed_form():
    """SPEC.md l.213-214 worked example; tests/golden/tls_2x2.txt."""
    A = np.array([[2.0], [0.0]])
    b = np.array([1.0, 1.0])
    ex = exact.tls_svd(A, b)
    assert ex.sigma ** 2 == pytest.approx(3 - math.sqrt(5), rel=1e-14)
    assert ex.x[0] == pytest.approx((math.sqrt(5) - 1) / 2, rel=1e-14)


def test_delta_matrix_secular_equation():
    """PAPER.md Example 2 matrix (l.502-531, delta = 1e-2, b = ones).  Its columns are
    orthogonal with norms (d, d, 1, 1), so [A,b]^T[A,b] is an arrow matrix and the
    smallest eigenvalue lam solves sum c_i^2/(s_i^2 - lam) = b^T b - lam with
    c = A^T b = (d, d, 1, 1), s^2 = (d^2, d^2, 1, 1); x_TLS,i = c_i/(s_i^2 - lam).
    Root by bisection on (0, d^2): independent of any SVD."""
    d = 1e-2
    A = _delta_matrix(d)
    b = np.ones(9)
    c = A.T @ b
    s2 = np.sum(A * A, axis=0)
    F = lambda lam: np.sum(c * c / (s2 - lam)) - (b @ b - lam)
    lo, hi = 0.0, d * d * (1 - 1e-15)
    assert F(lo) < 0 < F(hi)
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if F(mid) < 0:
            lo = mid
        else:
            hi = mid
    lam = 0.5 * (lo + hi)
    ex = exact.tls_svd(A, b)
    assert ex.sigma ** 2 == pytest.approx(lam, rel=1e-9)
    np.testing.assert_allclose(ex.x, c / (s2 - lam), rtol=1e-8)


def test_rayleigh_invariant_and_two_routes():
    """||[A,b][x;-1]||^2/(1+||x||^2) = sigma_{n+1}^2 at x_TLS;
    SVD route (gesdd) equals the QR->SVD route used for tall configs."""
    P = tlsgen.config("cfg1")
    ex = exact.tls_svd(P.A, P.b)
    ex2 = exact.tls_qr_svd(P.A, P.b)
    assert exact.rayleigh_sigma2(P.A, P.b, ex.x) == pytest.approx(ex.sigma ** 2, rel=1e-12)
    assert ex2.sigma == pytest.approx(ex.sigma, rel=1e-13)
    np.testing.assert_allclose(ex2.x, ex.x, rtol=1e-12)
    # x_TLS minimises the Rayleigh quotient: random perturbations increase it
    rng = np.random.default_rng(0)
    for _ in range(20):
        y = ex.x + 1e-3 * rng.standard_normal(ex.x.shape)
        assert exact.rayleigh_sigma2(P.A, P.b, y) > ex.sigma ** 2


def test_arrow_model_matches_svd():
    """Reduced model K = [[diag(s), c], [0, rho]] with c = U^T b, rho = ||b - U c||."""
    for name in ("cfg1", "cfg2w"):
        P = tlsgen.config(name, m=1024 if name == "cfg2w" else 200, n=64 if name == "cfg2w" else 20)
        c = P.U.T @ P.b
        rho = np.linalg.norm(P.b - P.U @ c)
        ex_a = exact.tls_arrow(P.s, P.V, c, rho)
        ex_s = exact.tls_svd(P.A, P.b)
        assert ex_a.sigma == pytest.approx(ex_s.sigma, rel=1e-10)
        np.testing.assert_allclose(ex_a.x, ex_s.x, rtol=1e-9)
        assert ex_a.unique and ex_s.unique


def test_literal_cfg2_nearly_nongeneric():
    """Reading R8: literal cfg2 has 1 - sigma^2/sigma'^2 ~ 5e-4 and
    kappa_TLS >~ 1e6, the twin cfg2w has kappa_TLS ~ 1e3."""
    P = tlsgen.config("cfg2")
    Pw = tlsgen.config("cfg2w")
    e, ew = exact.tls_svd(P.A, P.b), exact.tls_svd(Pw.A, Pw.b)
    assert e.kappa_tls > 1e6 and ew.kappa_tls < 1e4
    cons = exact.constraints(P.A, e)
    assert cons["gap"] < 1e-2


def test_constraint_report_closed_forms():
    """constraint_report (§3.1 D1-D8) on cases with closed forms: orthogonal
    columns of different norms give H = I, so D6 = 1/((2 + n)(n + 1)); D3/D5/D1/D2/D4 are
    the printed powers of kappa; D7 solves c m n u/(1 - c m n u) = gap/(sqrt(m) kappa_F)
    exactly at its value; D8 = constr2 of exact.constraints."""
    m, n = 50, 6
    Q, _ = np.linalg.qr(np.random.default_rng(1).standard_normal((m, n)))
    A = Q * np.array([1.0, 2.0, 4.0, 8.0, 16.0, 32.0])
    assert exact.lam_min_H(A) == pytest.approx(1.0, rel=1e-12)
    b = A @ np.ones(n) + 0.1 * np.random.default_rng(2).standard_normal(m)
    ex = exact.tls_svd(A, b)
    sA = np.linalg.svd(A, compute_uv=False)
    r = exact.constraint_report(m, n, sA, ex.sigma, float(np.linalg.norm(A)), exact.lam_min_H(A))
    kap = 32.0
    assert r["kappa"] == pytest.approx(kap, rel=1e-12)
    assert r["D3"] == pytest.approx(1 / kap) and r["D5"] == pytest.approx(1 / kap ** 2)
    assert r["D1"] == pytest.approx(1 / (m * n ** 1.5 * kap)) and r["D2"] == pytest.approx(1 / (m ** 0.5 * n ** 0.75 * kap))
    assert r["D4"] == pytest.approx(1 / (20 * n ** 1.5 * kap ** 2))
    assert r["D6"] == pytest.approx(1.0 / ((2.0 + n) * (n + 1)), rel=1e-12)
    u = r["D7"]
    gmn = m * n * u / (1 - m * n * u)
    assert np.sqrt(m) * gmn * r["kappa_F"] == pytest.approx(r["gap"], rel=1e-12)
    assert r["D8"] == pytest.approx(exact.constraints(A, ex)["constr2"], rel=1e-14)
