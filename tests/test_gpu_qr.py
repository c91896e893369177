"""GPU parity of the Householder-QR preconditioner in u_f (PAPER.md
l.215-218, l.231; readings R25-R27) against oracle/qr.py through the C ABI.

Both sides round every elementwise operation to u_f at the same points (pinned exactly by
test_oracle_qr.test_householder_rounding_points_exact) and take the same sign decisions; only
the fp64 inner products (x^T x, v^T W) are summed in another order before their single
rounding to u_f, which changes a rounded value only when the fp64 sum lies within its own
rounding error (~1e-16 relative) of a u_f rounding boundary.  So
  - D and ||A||_F^2: bit-exact / 1e-14;
  - R~ (u_f = fp16 / bf16 / fp32): entrywise in u_f ulps -- bit-identical on >= 99% of the
    entries and within 2 ulps everywhere (_assert_entrywise);  u_f = fp64: the summation order
    itself is the rounding, so 1e-12 kappa(Ah) relative (normwise) instead;
  - a solve with the GPU's QR R~: the north_star tolerances against the oracle run on the
    same R~ (x 1e-9, sigma 1e-12, same RQI count, PCG counts equal) and against the SVD.
"""
import numpy as np
import pytest
import torch

import tlsgen
from oracle import exact, rqi
from oracle.rounding import round_to, unit_roundoff

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def T():
    from paper_2305_19028_b200 import tlsrqi
    tlsrqi.lib()
    return tlsrqi


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def _mat(T, A):
    """tls_matrix_t of A with an even leading dimension (the ABI's dense layout); returns the
    device tensor too, which must stay alive while the matrix is used."""
    m, n = A.shape
    Ap = np.zeros((m, n + (n & 1)))
    Ap[:, :n] = A
    t = dev(Ap)
    return T.matrix(t, n=n), t


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def _ordered(x, fmt):
    """u_f values -> integers whose differences count u_f ulps (sign-magnitude folded)."""
    x = np.asarray(x, dtype=np.float64)
    if fmt == "fp16":
        b = x.astype(np.float16).view(np.int16).astype(np.int64)
        return np.where(b < 0, -(b & 0x7FFF), b)
    b = x.astype(np.float32).view(np.int32).astype(np.int64)
    if fmt == "bf16":
        b = b >> 16
        return np.where(b < 0, -(b & 0x7FFF), b)
    return np.where(b < 0, -(b & 0x7FFFFFFF), b)


def _assert_entrywise(Rt, Ro, fmt, frac_equal=0.99, max_ulps=2):
    """GPU R~ vs oracle R~ entry by entry: identical bits on >= frac_equal of the stored
    (upper) entries and at most max_ulps u_f ulps apart elsewhere; u_f = fp64: normwise."""
    iu = np.triu_indices(Rt.shape[0])
    if fmt == "fp64":
        assert _rel(Rt, Ro) <= 1e-12 * max(1.0, np.linalg.cond(Ro))
        return
    a, b = Rt[iu], Ro[iu]
    same = np.mean(a.view(np.uint64) == b.view(np.uint64))
    ulps = np.abs(_ordered(a, fmt) - _ordered(b, fmt))
    assert same >= frac_equal and ulps.max() <= max_ulps, (same, int(ulps.max()))


def _problem(m, n, kappa, seed, spread=True):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((m, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = np.logspace(0, -np.log10(kappa), n)
    A = (U * s) @ V.T
    # column scales spread over several binades so that D is not the identity
    if spread:
        A = A * np.exp2(rng.integers(-6, 7, n))[None, :]
    x = rng.standard_normal(n)
    b = A @ x + 1e-3 * rng.standard_normal(m) * np.linalg.norm(A @ x) / np.sqrt(m)
    return A, b


CASES = [  # (m, n, kappa, u_f): tiles of 256 columns per thread sweep, ragged tails, all formats
    (200, 20, 1e2, "fp16"), (333, 47, 1e2, "bf16"), (777, 67, 1e3, "fp32"), (257, 31, 1e3, "fp64"),
    (600, 300, 1e2, "fp16"), (1100, 530, 1e2, "bf16"), (1100, 530, 1e2, "fp16"), (1500, 700, 1e2, "fp16")]


@pytest.mark.parametrize("m,n,kappa,fmt", CASES)
def test_qr_factor_parity(T, m, n, kappa, fmt):
    A, _ = _problem(m, n, kappa, seed=m + n)
    pc = rqi.factor_precond_qr(A, fmt)
    assert pc.status == rqi.OK
    M, keep = _mat(T, A)
    rc, R, info = T.tls_factor_precond_qr(M, fmt)
    assert rc == 0 and R is not None
    Rt, d, nrm = T.tls_precond_export(R)
    assert np.array_equal(d, pc.d)
    assert nrm == pytest.approx(pc.normA2, rel=1e-14)
    assert np.array_equal(np.tril(Rt, -1), np.zeros_like(Rt))
    assert np.all(np.diag(Rt) > 0)
    assert np.array_equal(round_to(Rt, fmt), Rt)                 # stored in u_f
    _assert_entrywise(Rt, pc.Rt, fmt)


@pytest.mark.parametrize("m,n,kappa,fmt", [(200, 20, 1e2, "fp16"), (777, 67, 1e3, "bf16"), (5000, 1100, 1e2, "fp16"),
                                           (1100, 530, 1e2, "fp16")])
def test_qr_solve_parity(T, m, n, kappa, fmt):
    """RQI-PCGTLS-MP preconditioned by the GPU's QR R~ against the oracle on the same R~."""
    A, b = _problem(m, n, kappa, seed=7 * m + n, spread=False)   # sigma_n(A) >> sigma_{n+1}: a TLS solution exists
    M, keep = _mat(T, A)
    rc, R, _ = T.tls_factor_precond_qr(M, fmt)
    assert rc == 0
    rc, x, sig, info = T.tls_rqi_pcgtls(M, dev(b), R)
    Rt, d, nrm = T.tls_precond_export(R)
    if m * n * n <= 4e8:                    # the oracle's u_f QR costs O(m n^2) numpy passes
        _assert_entrywise(Rt, rqi.factor_precond_qr(A, fmt).Rt, fmt)
    res = rqi.rqi_pcgtls_mp(A, b, rqi.Precond(Rt, d, fmt, nrm))
    ex = exact.tls_svd(A, b)
    assert info["status"] == res.status == rqi.OK
    assert info["rqi_iters"] == res.rqi_iters
    assert info["pcg_iters"] == [tuple(p) for p in res.pcg_iters]
    assert _rel(x.cpu().numpy(), res.x) <= 1e-9
    assert abs(sig - res.sigma) / res.sigma <= 1e-12
    assert _rel(x.cpu().numpy(), ex.x) <= 1e-9


def test_qr_cfg1_paper_workload(T):
    """cfg1 (BASELINE configs[0]) with the paper's preferred preconditioner, u_f = fp16."""
    P = tlsgen.config("cfg1")
    M = T.matrix(dev(P.A))
    rc, R, _ = T.tls_factor_precond_qr(M, "fp16")
    assert rc == 0
    Rt, d, nrm = T.tls_precond_export(R)
    pc = rqi.factor_precond_qr(P.A, "fp16")
    _assert_entrywise(Rt, pc.Rt, "fp16")
    rc, x, sig, info = T.tls_rqi_pcgtls(M, dev(P.b), R)
    ex = exact.tls_svd(P.A, P.b)
    assert _rel(x.cpu().numpy(), ex.x) <= 1e-9
    assert abs(sig - ex.sigma) / ex.sigma <= 1e-11


def test_qr_zero_column_breakdown(T):
    """Column 1 equals 2 x column 0 = 2 e_0: after the power-of-two scaling both are e_0, the
    first reflector maps column 1 to -e_0 exactly, and column 1 is exactly zero below the
    diagonal.  Both sides report the 1-based pivot 2."""
    rng = np.random.default_rng(3)
    A = rng.standard_normal((64, 8))
    A[:, 0] = 0.0
    A[0, 0] = 1.0
    A[:, 1] = 2.0 * A[:, 0]
    for fmt in ("fp16", "fp32", "fp64"):
        pc = rqi.factor_precond_qr(A, fmt)
        assert pc.status == rqi.CHOL_BREAKDOWN and pc.chol_pivot == 2
        rc, R, info = T.tls_factor_precond_qr(T.matrix(dev(A)), fmt)
        assert R is None
        assert rc == rqi.CHOL_BREAKDOWN
        assert info["chol_pivot"] == pc.chol_pivot


def test_qr_refuses_csr_and_reports_workspace(T):
    A, _ = _problem(64, 8, 10.0, seed=1)
    M = T.matrix(dev(A))
    assert T.lib().tls_qr_workspace_size(M, 0, 1) >= 64 * 8 * 4
    assert T.lib().tls_qr_workspace_size(M, 0, 2) > T.lib().tls_qr_workspace_size(M, 0, 1)   # + the TSQR stack
    with pytest.raises(T.TlsError):
        T.tls_factor_precond_qr(M, "fp16", ws=torch.empty(16, dtype=torch.uint8, device="cuda"))


@pytest.mark.parametrize("name", tlsgen.PAPER_PROBLEMS)
@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
def test_paper_sec4_problems_qr(T, name, fmt):
    """The paper's §4 problems with the QR preconditioner it prefers (E5
    compares it with the Cholesky one): the GPU's QR R~ against the oracle's, and the solve
    on the GPU's R~ against the oracle on the same R~ (PCG counts within the north_star's +-2)."""
    P = tlsgen.paper_problem(name)
    M = T.matrix(T.dense_operand(dev(P.A)), n=P.n)
    pc = rqi.factor_precond_qr(P.A, fmt)
    rc, R, finfo = T.tls_factor_precond_qr(M, fmt)
    assert rc == pc.status
    if rc != 0:
        assert finfo["chol_pivot"] == pc.chol_pivot
        return
    Rt, d, nrm = T.tls_precond_export(R)
    _assert_entrywise(Rt, pc.Rt, fmt)
    rc, x, sig, info = T.tls_rqi_pcgtls(M, dev(P.b), R)
    res = rqi.rqi_pcgtls_mp(P.A, P.b, rqi.Precond(Rt, d, fmt, nrm))
    assert info["status"] == res.status
    assert info["rqi_iters"] == res.rqi_iters
    assert len(info["pcg_iters"]) == len(res.pcg_iters)
    for a, b in zip(info["pcg_iters"], res.pcg_iters):
        assert abs(a[0] - b[0]) <= 2 and abs(a[1] - b[1]) <= 2
    if res.status == rqi.OK:
        ex = exact.tls_svd(P.A, P.b)
        assert _rel(x.cpu().numpy(), res.x) <= 1e-9
        assert abs(sig - res.sigma) / res.sigma <= 1e-12
        assert _rel(x.cpu().numpy(), ex.x) <= 1e-9


@pytest.mark.parametrize("leaves,m,n,fmt", [(2, 200, 20, "fp16"), (3, 777, 67, "bf16"), (4, 1200, 270, "fp16"),
                                            (2, 300, 31, "fp64")])
def test_qr_tsqr_leaves(T, monkeypatch, leaves, m, n, fmt):
    """TSQR (R26) through the same code path a row-sharded factorization takes, on one GPU:
    TLS_QR_LEAVES = k splits the rows into k leaves.  Against the oracle's tsqr_r on the same
    leaves (bounds as in test_qr_factor_parity, two levels), then a solve on that R~."""
    from oracle.qr import even_row_blocks
    monkeypatch.setenv("TLS_QR_LEAVES", str(leaves))
    A, b = _problem(m, n, 1e2, seed=3 * m + n, spread=False)
    M, keep = _mat(T, A)
    rc, R, info = T.tls_factor_precond_qr(M, fmt)
    assert rc == 0
    pc = rqi.factor_precond_qr(A, fmt, row_blocks=even_row_blocks(m, leaves))
    Rt, d, nrm = T.tls_precond_export(R)
    assert np.array_equal(d, pc.d)
    assert np.all(np.diag(Rt) > 0) and np.array_equal(round_to(Rt, fmt), Rt)
    _assert_entrywise(Rt, pc.Rt, fmt)
    rc, x, sig, info = T.tls_rqi_pcgtls(M, dev(b), R)
    res = rqi.rqi_pcgtls_mp(A, b, rqi.Precond(Rt, d, fmt, nrm))
    assert info["status"] == res.status == rqi.OK
    assert info["rqi_iters"] == res.rqi_iters
    assert info["pcg_iters"] == [tuple(p) for p in res.pcg_iters]
    assert _rel(x.cpu().numpy(), res.x) <= 1e-9
    assert abs(sig - res.sigma) / res.sigma <= 1e-12


@pytest.mark.parametrize("leaves,m,n", [(3, 14209, 16), (2, 9473, 16)])
def test_qr_tsqr_leaf_partials_sizing(T, monkeypatch, leaves, m, n):
    """qr_rows_per_cta is not monotone in m -- 14209 rows in 3 leaves of 4736/4737
    rows use 148/148/144 update CTAs against 147 for 14209 rows, 9473 in 2 leaves 148 vs 146.
    The partials buffer is sized for every leaf; R~ equals the oracle's tsqr_r entrywise."""
    from oracle.qr import even_row_blocks
    monkeypatch.setenv("TLS_QR_LEAVES", str(leaves))
    A, b = _problem(m, n, 1e2, seed=m, spread=True)
    M, keep = _mat(T, A)
    rc, R, info = T.tls_factor_precond_qr(M, "fp16")
    assert rc == 0
    Rt, d, nrm = T.tls_precond_export(R)
    pc = rqi.factor_precond_qr(A, "fp16", row_blocks=even_row_blocks(m, leaves))
    _assert_entrywise(Rt, pc.Rt, "fp16")


@pytest.mark.parametrize("fmt", ["fp16", "fp64"])
def test_qr_tsqr_leaf_vanishing_column(T, monkeypatch, fmt):
    """a column that is zero on one leaf's rows of a full-rank A is not a rank
    deficiency -- the leaf takes the identity reflector (R26) and the factorization succeeds
    with the oracle's tsqr_r R~; a column zero on every row is still CHOL_BREAKDOWN."""
    from oracle.qr import even_row_blocks
    monkeypatch.setenv("TLS_QR_LEAVES", "3")
    A, b = _problem(900, 24, 1e2, seed=17, spread=False)
    A[:300, 5] = 0.0
    M, keep = _mat(T, A)
    rc, R, info = T.tls_factor_precond_qr(M, fmt)
    pc = rqi.factor_precond_qr(A, fmt, row_blocks=even_row_blocks(900, 3))
    assert rc == pc.status == 0
    Rt, d, nrm = T.tls_precond_export(R)
    _assert_entrywise(Rt, pc.Rt, fmt)
    A[:, 5] = 0.0
    A[0, 5] = 0.0
    M2, keep2 = _mat(T, A)
    with pytest.raises(T.TlsError):       # a zero column of A itself is an argument error (rank deficient)
        T.tls_factor_precond_qr(M2, fmt)


def test_qr_tsqr_leaf_too_short(T, monkeypatch):
    monkeypatch.setenv("TLS_QR_LEAVES", "8")
    A, _ = _problem(100, 20, 10.0, seed=2)
    M, keep = _mat(T, A)
    with pytest.raises(T.TlsError):
        T.tls_factor_precond_qr(M, "fp16")


@pytest.mark.parametrize("m,n,fmt", [(5, 1, "fp16"), (2300, 2100, "fp16"), (4200, 4096, "bf16")])
def test_qr_extreme_widths(T, m, n, fmt):
    """n = 1 (no update pass at all) and n > 2048 (16 columns per thread; n = 4096 is the
    largest dense n): the R~ the GPU returns is a QR factor of fl(A D^{-1}) within the pinned
    backward-error bound, upper with a positive diagonal, in u_f; then a solve on it matches
    the oracle run on the same R~."""
    A, b = _problem(m, n, 10.0, seed=m + 7 * n, spread=False)
    M, keep = _mat(T, A)
    rc, R, _ = T.tls_factor_precond_qr(M, fmt)
    assert rc == 0
    Rt, d, nrm = T.tls_precond_export(R)
    assert np.array_equal(np.tril(Rt, -1), np.zeros_like(Rt)) and np.all(np.diag(Rt) > 0)
    assert np.array_equal(round_to(Rt, fmt), Rt)
    Ah = round_to(A / d, fmt)
    if m * n * n <= 4e8:
        _assert_entrywise(Rt, rqi.factor_precond_qr(A, fmt).Rt, fmt)
    else:                                   # backward error of the GPU's R~ (probabilistic form, c = 2)
        u = unit_roundoff(fmt)
        assert np.linalg.norm(Rt.T @ Rt - Ah.T @ Ah) <= 2 * np.sqrt(m) * n ** 0.75 * u * np.linalg.norm(Ah) ** 2
    if n == 1:
        assert Rt[0, 0] == pytest.approx(np.linalg.norm(Ah), rel=2 * unit_roundoff(fmt))
        return
    rc, x, sig, info = T.tls_rqi_pcgtls(M, dev(b), R)
    res = rqi.rqi_pcgtls_mp(A, b, rqi.Precond(Rt, d, fmt, nrm))
    assert info["status"] == res.status
    assert info["rqi_iters"] == res.rqi_iters
    if res.status == rqi.OK:
        assert _rel(x.cpu().numpy(), res.x) <= 1e-9
        assert abs(sig - res.sigma) / res.sigma <= 1e-12


def test_qr_norm_scaling_keeps_fp16_in_range(T):
    """A tall column of 70000 entries in [1/2, 1): under round 1's max-based D its x^T x
    (> 65504) overflowed fp16 when rounded (TLS_RANGE).  The paper's
    D = diag(A^T A)^{1/2} rounded to powers of two (R27) scales every column to
    a norm in [2^-1/2, 2^1/2), so fp16 factors it -- bit for bit like the oracle -- and so does
    bf16."""
    rng = np.random.default_rng(0)
    A = rng.uniform(0.5, 1.0, (70000, 4))
    M, keep = _mat(T, A)
    for fmt in ("fp16", "bf16"):
        pc = rqi.factor_precond_qr(A, fmt)
        assert pc.status == rqi.OK
        rc, R, info = T.tls_factor_precond_qr(M, fmt)
        assert rc == 0
        Rt, d, nrm = T.tls_precond_export(R)
        assert np.array_equal(d, pc.d)
        _assert_entrywise(Rt, pc.Rt, fmt)
