"""Pins of oracle/qr.py (Householder QR in u_q; SURVEY §8(f) NEXT-2 groundwork):
SPEC.md's worked examples, LAPACK agreement in fp64, the Gram residual bound in low
precision, and the paper's point that QR depends on kappa where the Gram Cholesky
depends on kappa^2."""
import numpy as np
import pytest

from oracle.qr import householder_qr_r
from oracle.rounding import round_to, unit_roundoff


def test_spec_examples():
    """SPEC.md householder_qr examples: QR(I_n) = I_n; QR([3;4]) = [5]."""
    assert np.array_equal(householder_qr_r(np.eye(5), "fp64"), np.eye(5))
    assert householder_qr_r(np.array([[3.0], [4.0]]), "fp64")[0, 0] == 5.0


def test_fp64_matches_lapack():
    """In fp64 the R factor equals LAPACK's (numpy.linalg.qr) up to row signs."""
    rng = np.random.default_rng(4)
    A = rng.standard_normal((20, 10))
    R = householder_qr_r(A, "fp64")
    Rl = np.linalg.qr(A, mode="r")
    Rl = Rl * np.where(np.diag(Rl) < 0, -1.0, 1.0)[:, None]
    assert np.allclose(R, Rl, rtol=1e-13, atol=1e-13)
    assert np.all(np.diag(R) >= 0)


@pytest.mark.parametrize("fmt", ["fp16", "bf16", "fp32"])
def test_gram_residual_bound(fmt):
    """SPEC.md invariant 'QR residual <= 10 m n u' in Gram form (Q is not formed):
    ||R^T R - Ah^T Ah||_F <= 10 m n u ||Ah||_F^2 with Ah = fl(A)."""
    rng = np.random.default_rng(5)
    m, n = 60, 12
    A = round_to(rng.standard_normal((m, n)), fmt)
    R = householder_qr_r(A, fmt)
    u = unit_roundoff(fmt)
    assert np.linalg.norm(R.T @ R - A.T @ A) <= 10 * m * n * u * np.linalg.norm(A) ** 2


def test_qr_needs_kappa_where_cholesky_needs_kappa_squared():
    """PAPER.md l.276-297 / SPEC.md cholesky_scaled example: with kappa(A)^2 > 1/u_fp16
    but u_fp16 kappa(A) < 1, the Cholesky of the fp16-rounded Gram fl(A^T A) (the unscaled
    pathway) breaks down while the fp16 Householder R is nonsingular and preconditions A
    (kappa(A R^{-1}) small)."""
    rng = np.random.default_rng(6)
    m, n = 80, 10
    U, _ = np.linalg.qr(rng.standard_normal((m, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)))
    kappa = 300.0                      # kappa^2 = 9e4 > 1/u = 2048; u kappa = 0.15
    A = (U * np.logspace(0, -np.log10(kappa), n)) @ V.T
    G16 = round_to(round_to(A, "fp16").T @ round_to(A, "fp16"), "fp16")
    with pytest.raises(np.linalg.LinAlgError):
        np.linalg.cholesky(G16)
    R = householder_qr_r(A, "fp16")
    assert np.min(np.abs(np.diag(R))) > 0
    assert np.linalg.cond(A @ np.linalg.inv(R)) < 10.0


@pytest.mark.parametrize("name", ["cfg1", "random", "vanhuffel", "toeplitz"])
def test_rqi_with_qr_preconditioner(name):
    """RQI-PCGTLS-MP with the paper's own preconditioner (fp16 Householder R, PAPER.md
    l.231) reaches the SVD's x and sigma like the Cholesky route does."""
    import tlsgen
    from oracle import exact, rqi
    P = tlsgen.config(name) if name.startswith("cfg") else tlsgen.paper_problem(name)
    ex = exact.tls_svd(P.A, P.b)
    pc = rqi.factor_precond_qr(P.A, "fp16")
    assert pc.status == rqi.OK
    r = rqi.rqi_pcgtls_mp(P.A, P.b, pc)
    assert r.status == rqi.OK
    assert np.linalg.norm(r.x - ex.x) / np.linalg.norm(ex.x) <= 1e-12
    assert abs(r.sigma - ex.sigma) / ex.sigma <= 1e-12


def test_zero_column_reports_its_pivot():
    """Column 1 = 2 x column 0 = 2 e_0: the first reflector (sigma = 1, alpha = -1, v = 2 e_0,
    beta = 1/2) maps the scaled column 1 (= e_0) to -e_0 exactly, so column 1 vanishes below
    its diagonal: CHOL_BREAKDOWN with the 1-based pivot 2 in every format."""
    from oracle import rqi
    from oracle.qr import ZeroColumn, householder_qr_r
    rng = np.random.default_rng(3)
    A = rng.standard_normal((64, 8))
    A[:, 0] = 0.0
    A[0, 0] = 1.0
    A[:, 1] = 2.0 * A[:, 0]
    for fmt in ("fp16", "bf16", "fp32", "fp64"):
        with pytest.raises(ZeroColumn) as e:
            householder_qr_r(A / np.array([1.0, 2.0] + [1.0] * 6), fmt)
        assert e.value.col == 1
        pc = rqi.factor_precond_qr(A, fmt)
        assert pc.status == rqi.CHOL_BREAKDOWN and pc.chol_pivot == 2


def test_tsqr_fp64_equals_lapack_r():
    """TSQR (R26) in fp64: the R of the stacked leaf R's is LAPACK's R of the whole A up to
    row signs (A = diag(Q_b)[R_1; ...; R_B], [R_1; ...; R_B] = Q'R), for 1, 2, 3 and 5 leaves;
    a dropped or duplicated leaf changes R^T R = A^T A and fails."""
    from oracle.qr import even_row_blocks, tsqr_r
    rng = np.random.default_rng(11)
    A = rng.standard_normal((97, 9))
    R0 = np.linalg.qr(A, mode="r")
    R0 = R0 * np.where(np.diag(R0) < 0, -1.0, 1.0)[:, None]
    for k in (1, 2, 3, 5):
        R = tsqr_r(A, even_row_blocks(97, k), "fp64")
        assert np.max(np.abs(R - R0)) <= 1e-13 * np.max(np.abs(R0))
    # the leaves cover the rows exactly once
    for m, k in ((97, 5), (4096, 3), (10, 10)):
        bl = even_row_blocks(m, k)
        assert bl[0][0] == 0 and bl[-1][1] == m and all(a[1] == b[0] for a, b in zip(bl, bl[1:]))


@pytest.mark.parametrize("fmt", ["fp16", "bf16", "fp32"])
def test_tsqr_backward_error_bound(fmt):
    """Two levels of Householder QR in fmt: ||R^T R - Ah^T Ah||_F <= 2 x 10 m n u ||Ah||_F^2
    (each level's Gram residual bound, the leaf one applied block by block)."""
    from oracle.qr import even_row_blocks, tsqr_r
    rng = np.random.default_rng(5)
    m, n = 300, 12
    A = round_to(rng.standard_normal((m, n)) * np.logspace(0, -1, n)[None, :], fmt)
    R = tsqr_r(A, even_row_blocks(m, 3), fmt)
    u = unit_roundoff(fmt)
    assert np.all(np.diag(R) > 0)
    assert np.linalg.norm(R.T @ R - A.T @ A) <= 2 * 10 * m * n * u * np.linalg.norm(A) ** 2
