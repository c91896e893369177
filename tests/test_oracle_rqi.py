"""Pins for oracle/rqi.py (Alg. 3 PCGTLS, Alg. 4 RQI-PCGTLS-MP, scaled Cholesky).

Each test checks the oracle against something other than itself: a different
LAPACK route, a closed form, exact integer arithmetic, an independent model of
Alg. 2 in the singular-vector basis, or the paper's printed op counts."""
import math

import numpy as np
import pytest
import scipy.sparse

import tlsgen
from oracle import exact, perfmodel, rqi
from oracle.rounding import round_to


def _small(m=300, n=24, kappa=1e2, eps=1e-4, seed=11, twin=False):
    return tlsgen.dense_problem(m, n, kappa, eps, seed, twin=twin)


# ----------------------------------------------------------------------------- scaling / Gram
def test_column_scaling_powers_of_two():
    P = _small()
    d, normA2 = rqi.column_scaling(P.A)
    m2, e = np.frexp(d)
    assert np.all(m2 == 0.5)                                # exact powers of two
    amax = np.max(np.abs(P.A / d), axis=0)
    assert np.all((amax >= 1) & (amax < 2))
    assert normA2 == pytest.approx(np.linalg.norm(P.A) ** 2, rel=1e-14)


def test_gram_integer_inputs_exact():
    """Small integers are exact in fp16 and all partial sums stay exact in fp32,
    so the emulated Gram equals the exact integer Gram (scaled by d d^T)."""
    rng = np.random.default_rng(0)
    A = rng.integers(-7, 8, size=(5000, 12)).astype(np.float64)
    A[0] = 7.0
    d, _ = rqi.column_scaling(A)
    for fmt in ("fp16", "bf16", "fp32", "fp64"):
        G = rqi.gram_uf(A, d, fmt, K_t=2048)
        exactG = (A.T.astype(np.int64) @ A.astype(np.int64)).astype(np.float64) / np.outer(d, d)
        assert np.array_equal(G, exactG)


def test_gram_error_bound_and_chunking():
    P = tlsgen.config("cfg2w", m=8192, n=64)
    d, _ = rqi.column_scaling(P.A)
    for fmt in ("fp16", "bf16"):
        Ah = round_to(P.A / d, fmt)
        G64 = Ah.T @ Ah
        G = rqi.gram_uf(P.A, d, fmt, K_t=2048)
        B = rqi.gram_exact_bound(P.A, d, fmt, K_t=2048)
        assert np.all(np.abs(G - G64) <= B)
        assert np.max(np.abs(G - G64)) > 0                  # fp32 accumulation is visible
        # one row per chunk: fp32 products exact -> fp64 sum of exact products
        G1 = rqi.gram_uf(P.A[:512], d, fmt, K_t=1)
        np.testing.assert_allclose(G1, Ah[:512].T @ Ah[:512], rtol=1e-13, atol=1e-12)


# ----------------------------------------------------------------------------- Cholesky
def test_cholesky_reconstruction_and_qr_route():
    P = _small(m=2000, n=40, kappa=1e2)
    pc = rqi.factor_precond(P.A, "fp64", keep=True)
    assert pc.status == rqi.OK
    np.testing.assert_allclose(pc.R.T @ pc.R, pc.G, rtol=1e-13, atol=1e-10 * np.abs(pc.G).max())
    assert np.all(np.diag(pc.R) > 0)
    # R-factor of Householder QR of A D^-1 equals the Cholesky factor up to row signs
    Rq = np.linalg.qr(P.A / pc.d, mode="r")
    np.testing.assert_allclose(np.abs(Rq), np.abs(pc.R), rtol=1e-9, atol=1e-9 * np.abs(pc.R).max())
    # R~ is R rounded to u_f
    pc16 = rqi.factor_precond(P.A, "fp16", keep=True)
    assert np.array_equal(pc16.Rt, round_to(np.triu(pc16.R), "fp16"))


def test_cholesky_breakdown_index():
    """Exact arithmetic: 39 orthogonal 0/1 columns with four ones each (G_jj = 4,
    R_jj = 2 exactly) and column 40 = column 18, so the 40th pivot is exactly 0
    for every u_f and chunk size."""
    n = 40
    A = np.zeros((4 * (n - 1), n))
    for i in range(A.shape[0]):
        A[i, i % (n - 1)] = 1.0
    A[:, n - 1] = A[:, 17]
    for fmt in ("fp16", "bf16", "fp32", "fp64"):
        for K_t in (1, 64, 2048):
            pc = rqi.factor_precond(A, fmt, K_t)
            assert pc.status == rqi.CHOL_BREAKDOWN and pc.chol_pivot == n


def test_precond_solves_vs_dense_solve():
    P = _small()
    pc = rqi.factor_precond(P.A, "bf16")
    Pm = pc.Rt * pc.d[None, :]                              # P = R~ D
    y = np.random.default_rng(0).standard_normal(P.n)
    np.testing.assert_allclose(rqi.apply_Pinv(pc, y), np.linalg.solve(Pm, y), rtol=1e-10)
    np.testing.assert_allclose(rqi.apply_PinvT(pc, y), np.linalg.solve(Pm.T, y), rtol=1e-10)


# ----------------------------------------------------------------------------- PCGTLS
def test_pcgtls_identities():
    """f = 0 -> 0 iterations; sigma = 0 with an exact factor ->
    one iteration gives (A^T A)^{-1} f; l = n -> the direct solve."""
    P = _small(m=400, n=16)
    f = np.random.default_rng(1).standard_normal(P.n)
    pc64 = rqi.factor_precond(P.A, "fp64")
    r0 = rqi.pcgtls(P.A, pc64, 0.3, np.zeros(P.n), 5, 1e-14)
    assert r0.count == 0 and not np.any(r0.omega)
    r1 = rqi.pcgtls(P.A, pc64, 0.0, f, 5, 1e-10)
    assert r1.count == 1
    np.testing.assert_allclose(r1.omega, np.linalg.solve(P.A.T @ P.A, f), rtol=1e-10)
    sA = np.linalg.svd(P.A, compute_uv=False)
    sig2 = 0.5 * sA[-1] ** 2
    pc16 = rqi.factor_precond(P.A, "fp16")
    M = P.A.T @ P.A - sig2 * np.eye(P.n)
    for variant in ("A", "paper"):
        rn = rqi.pcgtls(P.A, pc16 if variant == "A" else pc64, sig2, f, P.n, 1e-15, variant)
        np.testing.assert_allclose(rn.omega, np.linalg.solve(M, f), rtol=1e-9)


def test_pcgtls_variants_agree_for_exact_factor():
    """Reading R1: with R~ = R (u_f = fp64) both operator forms are the same
    operator, so their iterates agree to ~kappa(A)^2 u."""
    P = _small(m=500, n=20, kappa=1e2)
    pc = rqi.factor_precond(P.A, "fp64")
    f = np.random.default_rng(2).standard_normal(P.n)
    sig2 = 0.3 * np.linalg.svd(P.A, compute_uv=False)[-1] ** 2
    for l in (1, 2, 3):
        a = rqi.pcgtls(P.A, pc, sig2, f, l, 0.0, "A")
        b = rqi.pcgtls(P.A, pc, sig2, f, l, 0.0, "paper")
        assert a.count == b.count == l
        np.testing.assert_allclose(a.omega, b.omega, rtol=1e-8)


def test_pcgtls_indefinite_breakdown():
    """sigma^2 above sigma'_n^2: A^T A - sigma^2 I is indefinite; a direction of
    negative curvature gives delta < 0 -> breakdown (spec rule, R3)."""
    P = _small(m=400, n=16)
    pc = rqi.factor_precond(P.A, "fp64")
    sA = np.linalg.svd(P.A, full_matrices=False)
    v_min = sA[2][-1]
    sig2 = 2.0 * sA[1][-1] ** 2
    r = rqi.pcgtls(P.A, pc, sig2, v_min, 5, 1e-14)
    assert r.breakdown and r.breakdown_j == 0 and r.delta_min < 0


def test_cgls_bootstrap_is_least_squares():
    P = _small(m=800, n=30, kappa=1e3)
    pc = rqi.factor_precond(P.A, "fp16")
    r = rqi.pcgtls(P.A, pc, 0.0, P.A.T @ P.b, 200, 1e-13)
    xls = np.linalg.lstsq(P.A, P.b, rcond=None)[0]
    np.testing.assert_allclose(r.omega, xls, rtol=1e-9)


# ----------------------------------------------------------------------------- RQI
def _diag_model_trace(s, c, rho, steps):
    """Alg. 2 with EXACT inner solves written in the right-singular basis
    y = V^T x of A = U diag(s) V^T (independent of the oracle's code):
    r = U(c - s y) + b_perp, A^T r = V(s (c - s y)), b^T r = c^T(c - s y) + rho^2,
    (A^T A - sig2 I) -> diag(s^2 - sig2)."""
    y = c / s                                          # x_LS
    e = c - s * y
    sig0 = (e @ e + rho * rho) / (1 + y @ y)
    y = y + sig0 * y / s ** 2                          # x_1 = x_0 + sig0 (A^TA)^-1 x_0
    out = []
    for _ in range(steps):
        e = c - s * y
        yy = y @ y
        sig2 = (e @ e + rho * rho) / (1 + yy)
        f = -(s * e) - sig2 * y
        g = -(c @ e + rho * rho) + sig2
        psi = math.sqrt((f @ f + g * g) / (yy + 1))
        out.append((sig2, psi))
        om = -f / (s * s - sig2)
        z = y + om
        beta = (z @ f - g) / (z @ y + 1)
        u = y / (s * s - sig2)
        y = z + beta * u
    return out


def test_rqi_matches_diagonal_exact_model():
    """with u_f = fp64 and inner solves run to tol (budget rule
    1), the oracle's sigma_k^2 and psi_k follow the exact-solve model step by step."""
    P = tlsgen.dense_problem(600, 12, 1e2, 1e-2, 21, twin=True)
    c = P.U.T @ P.b
    rho = np.linalg.norm(P.b - P.U @ c)
    pc = rqi.factor_precond(P.A, "fp64")
    opts = rqi.RqiOptions(budget_rule=1, tol_inner=1e-15, boot_tol=1e-15, polish=1)
    res = rqi.rqi_pcgtls_mp(P.A, P.b, pc, tol=1e-15, opts=opts)
    model = _diag_model_trace(P.s, c, rho, len(res.sigma2_trace))
    normAb2 = np.linalg.norm(P.A) ** 2 + P.b @ P.b
    checked = 0
    for k, ((s2m, psim), s2o, psio) in enumerate(zip(model, res.sigma2_trace, res.psi_trace)):
        assert s2o == pytest.approx(s2m, rel=1e-10)
        if psim > 1e-13 * normAb2:
            assert psio == pytest.approx(psim, rel=1e-3)
            checked += 1
    assert checked >= 2
    ex = exact.tls_svd(P.A, P.b)
    assert math.sqrt(res.sigma2_trace[-1]) == pytest.approx(ex.sigma, rel=1e-12)


def test_tau_identity():
    """with J z = A^T b, tau = b^T(b - A z) - rho = z^T f - g."""
    P = _small(m=300, n=10, kappa=1e1)
    x = np.random.default_rng(5).standard_normal(P.n)
    sig2, f, g, _ = rqi.newton_residual(P.A, P.b, x)
    J = P.A.T @ P.A - sig2 * np.eye(P.n)
    z = x + np.linalg.solve(J, -f)
    np.testing.assert_allclose(J @ z, P.A.T @ P.b, rtol=1e-9)
    tau1 = P.b @ (P.b - P.A @ z) - sig2
    tau2 = z @ f - g
    assert tau1 == pytest.approx(tau2, rel=1e-8)


def test_newton_residual_zero_at_solution():
    """at x_TLS, f = 0 and g = 0 (PAPER.md Eq. newton, l.109-119)."""
    P = _small()
    ex = exact.tls_svd(P.A, P.b)
    sig2, f, g, psi = rqi.newton_residual(P.A, P.b, ex.x)
    assert sig2 == pytest.approx(ex.sigma ** 2, rel=1e-12)
    assert psi < 1e-14 * (np.linalg.norm(P.A) ** 2)


@pytest.mark.parametrize("u_f", ["fp16", "bf16", "fp32", "fp64"])
def test_rqi_end_to_end_cfg1(u_f):
    P = tlsgen.config("cfg1")
    ex = exact.tls_svd(P.A, P.b)
    pc, res = rqi.solve(P.A, P.b, u_f)
    assert res.status == rqi.OK and res.termination == rqi.T_CONVERGED_TOL
    assert np.linalg.norm(res.x - ex.x) / np.linalg.norm(ex.x) < 1e-12
    assert abs(res.sigma - ex.sigma) / ex.sigma < 1e-12
    assert rqi.certify_sigma(P.A, P.b, res.x) == pytest.approx(ex.sigma, rel=1e-12)
    assert all(a == k + 1 and b == k + 1 for k, (a, b) in enumerate(res.pcg_iters, start=1))


def test_mixed_precision_needs_at_least_as_many_steps():
    """MP performs at least as many RQI steps as the
    uniform-precision run and reaches a similar limiting accuracy."""
    P = tlsgen.config("cfg2w", m=2048, n=256)
    ex = exact.tls_svd(P.A, P.b)
    K = {}
    for u_f in ("fp64", "fp16", "bf16"):
        _, res = rqi.solve(P.A, P.b, u_f)
        assert res.status == rqi.OK
        K[u_f] = res.rqi_iters
        assert np.linalg.norm(res.x - ex.x) / np.linalg.norm(ex.x) < 1e-10
    assert K["fp16"] >= K["fp64"] and K["bf16"] >= K["fp64"]


def test_literal_cfg2_breaks_down_at_first_step():
    """Reading R8: on literal cfg2, RQ(x_LS) lies far above sigma'_n^2, so the first
    PCG step meets negative curvature even with an exact factor."""
    P = tlsgen.config("cfg2")
    for u_f in ("fp64", "bf16"):
        _, res = rqi.solve(P.A, P.b, u_f)
        assert res.status == rqi.PCG_BREAKDOWN and res.breakdown_k == 1 and res.breakdown_j == 0


def test_sparse_matches_dense():
    Pc = tlsgen.csr_problem(m=3000, n=60, per_row=6, seed=7)
    As = scipy.sparse.csr_matrix((Pc.vals, Pc.colidx, Pc.rowptr), shape=(Pc.m, Pc.n))
    Ad = Pc.to_dense()
    assert np.all(np.diff(Pc.rowptr) == 7)
    for i in range(0, Pc.m, 397):                        # A20: distinct + fixed column
        cols = Pc.colidx[Pc.rowptr[i]:Pc.rowptr[i + 1]]
        assert len(set(cols)) == 7 and (i % Pc.n) in cols and np.all(np.diff(cols) > 0)
    pcs, rs = rqi.solve(As, Pc.b, "fp16")
    pcd, rd = rqi.solve(Ad, Pc.b, "fp16")
    # CSR Gram is the exact sum rounded once (R19), the dense one fp32 per 64-row
    # chunk (R11): R~ agrees to within one fp16 ulp entrywise
    ulp = np.spacing(np.abs(pcd.Rt).astype(np.float16)).astype(np.float64)
    assert np.all(np.abs(pcs.Rt - pcd.Rt) <= ulp)
    assert rs.rqi_iters == rd.rqi_iters
    np.testing.assert_allclose(rs.x, rd.x, rtol=1e-12)
    ex = exact.tls_svd(Ad, Pc.b)
    np.testing.assert_allclose(rs.x, ex.x, rtol=1e-11)


# ----------------------------------------------------------------------------- cost model
def test_cost_model_equals_sum_of_alg4_line_counts():
    """PAPER.md l.410-412 closed form == the per-line op counts printed in Alg. 4
    (l.227-255), PCGTLS performing exactly k+1 iterations at step k (l.405)."""
    for (m, n, r) in [(100, 60, 8), (30, 15, 5), (4096, 512, 7), (200, 20, 1)]:
        pre = (2*m*n + m) + (2*m + 2*n - 2) + (2*n*n) + (2*n)          # l.227-236 minus QR
        qr = 2*m*n*n - 2*n**3 / 3                                      # l.231-232
        per_k = lambda k: ((2*m*n + m) + (2*m + 2*n - 2) + (2*m*n + 2*n) + (2*m - 1)
                           + n + (4*n - 2) + (2*n))                    # l.238-255, u lines
        pcg_k = lambda k: 2 * ((k + 1) * (2*n*n + 14*n - 3) + (n*n + 2*n - 1))   # l.246-253
        tot_u = pre + sum(per_k(k) for k in range(1, r + 1))
        tot_p = sum(pcg_k(k) for k in range(1, r + 1))
        assert perfmodel.cost(m, n, r, 1, 0, 0) == tot_u
        assert perfmodel.cost(m, n, r, 0, 1, 0) == tot_p
        assert float(perfmodel.cost(m, n, r, 0, 0, 1)) == pytest.approx(qr, rel=1e-15)
    # "speedup never below 1" (l.449) and "up to 4x" (l.26)
    for (m, n, r) in [(10**6, 10**3, 5), (10**4, 10**4, 2000), (100, 60, 8)]:
        s = perfmodel.speedup(m, n, r)
        assert 1.0 <= s <= 4.0


# ----------------------------------------------------------------------------- CSR Gram (R19)
def _tiny_csr(m, n, per_row, seed, integer=False):
    rng = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    for i in range(m):
        c = np.sort(rng.choice(n, per_row, replace=False))
        v = rng.integers(-9, 10, per_row).astype(float) if integer else rng.standard_normal(per_row) * 10.0 ** rng.uniform(-3, 3)
        rows += [i] * per_row
        cols += list(c)
        vals += list(v)
    A = scipy.sparse.csr_matrix((vals, (rows, cols)), shape=(m, n))
    A.data[A.data == 0] = 1.0
    for j in range(n):                      # no empty column
        if A[:, j].nnz == 0:
            A[j % m, j] = 1.5
    return scipy.sparse.csr_matrix(A)


def test_csr_gram_fp16_is_exact_sum_rounded_once():
    """R19 pin: the fp16 CSR Gram equals the exact rational sum of the exact u_f
    products, rounded once (Fraction arithmetic, independent of the int64 split)."""
    from fractions import Fraction
    A = _tiny_csr(60, 7, 3, 11)
    d, _ = rqi.column_scaling(A)
    G = rqi.gram_uf(A, d, "fp16")
    Ah = A.toarray() / d[None, :]
    Ah = round_to(Ah, "fp16")
    for j in range(7):
        for k in range(7):
            ex = sum((Fraction(float(Ah[i, j])) * Fraction(float(Ah[i, k])) for i in range(60)), Fraction(0))
            assert G[j, k] == float(ex)


def test_csr_gram_integer_inputs_exact():
    A = _tiny_csr(400, 9, 4, 3, integer=True)
    d, _ = rqi.column_scaling(A)
    Ad = A.toarray()
    exactG = (Ad.T.astype(np.int64) @ Ad.astype(np.int64)).astype(np.float64) / np.outer(d, d)
    for fmt in ("fp16", "bf16", "fp32", "fp64"):
        assert np.array_equal(rqi.gram_uf(A, d, fmt), exactG)


def test_csr_gram_bf16_within_fp64_summation_bound():
    A = _tiny_csr(300, 12, 5, 5)
    d, _ = rqi.column_scaling(A)
    Ah = round_to(A.toarray() / d[None, :], "bf16")
    G = rqi.gram_uf(A, d, "bf16")
    bound = 300 * 2.0 ** -53 * (np.abs(Ah).T @ np.abs(Ah))
    assert np.all(np.abs(G - Ah.T @ Ah) <= 2 * bound)


# ----------------------------------------------------------------------------- u_p = fp32 (R23)
def test_operator_fp32_within_fp32_bound():
    """operator_fp32 (R23): v and t^T t lie within the closed-form fp32 accumulation
    bound around the exact product of the fp32-rounded data (gamma_k = k u/(1 - k u),
    u = 2^-24), and they are NOT the fp64 result (the arithmetic really is fp32)."""
    rng = np.random.default_rng(11)
    m, n = 3000, 300
    A = rng.standard_normal((m, n)) * np.logspace(0, -2, n)
    q = rng.standard_normal(n)
    A32 = A.astype(np.float32)
    tt, v = rqi.operator_fp32(A32, q)
    Ae = A32.astype(np.float64)
    qe = q.astype(np.float32).astype(np.float64)
    t_ex = Ae @ qe
    u = 2.0 ** -24
    g = lambda k: k * u / (1 - k * u)
    tb = g(n) * (np.abs(Ae) @ np.abs(qe))                    # |t32 - t_ex| bound
    t32 = (A32 @ q.astype(np.float32)).astype(np.float64)
    assert np.all(np.abs(t32 - t_ex) <= tb)
    vb = g(m) * (np.abs(Ae).T @ np.abs(t32)) + np.abs(Ae).T @ tb
    v_ex = Ae.T @ t_ex
    assert np.all(np.abs(v - v_ex) <= vb)
    assert abs(tt - float(t_ex @ t_ex)) <= 2.0 * float(np.abs(t_ex) @ tb) + 1e-300
    v64 = A.T @ (A @ q)
    assert np.max(np.abs(v - v64) / np.abs(v64).max()) > 1e-9      # fp32 arithmetic happened


@pytest.mark.parametrize("name", ["cfg1", "cfg2w", "random", "delta", "toeplitz", "vanhuffel"])
@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
def test_up_fp32_suffices(name, fmt):
    """with u = fp64, single precision for the PCG (u_p) 'was
    sufficient for all included examples': the same status and RQI count as u_p = fp64
    and the limiting accuracy of the SVD."""
    P = tlsgen.config(name) if name.startswith("cfg") else tlsgen.paper_problem(name)
    ex = exact.tls_svd(P.A, P.b)
    pc = rqi.factor_precond(P.A, fmt)
    r64 = rqi.rqi_pcgtls_mp(P.A, P.b, pc)
    r32 = rqi.rqi_pcgtls_mp(P.A, P.b, pc, opts=rqi.RqiOptions(u_p="fp32"))
    assert r32.status == r64.status == rqi.OK
    assert r32.rqi_iters == r64.rqi_iters
    assert np.linalg.norm(r32.x - ex.x) / np.linalg.norm(ex.x) <= 1e-12
    assert abs(r32.sigma - ex.sigma) / ex.sigma <= 1e-12


# ----------------------------------------------------------------------------- explicit inverse (R24)
def test_explicit_inverse_apply():
    """with_inverse (R24): W R~ = I, and P^{-1}, P^{-T} through W equal the substitutions
    to kappa(R~) u (the operator is the same linear map; only the rounding differs)."""
    P = tlsgen.config("cfg2w")
    pc = rqi.factor_precond(P.A, "bf16")
    pw = rqi.with_inverse(pc)
    n = pc.Rt.shape[0]
    assert np.allclose(pw.W @ pc.Rt, np.eye(n), atol=1e-12)
    assert np.array_equal(np.tril(pw.W, -1), np.zeros((n, n)))
    kap = np.linalg.cond(pc.Rt)
    y = np.random.default_rng(3).standard_normal(n)
    for f in (rqi.apply_Pinv, rqi.apply_PinvT):
        a, b = f(pc, y), f(pw, y)
        assert np.linalg.norm(a - b) <= 10 * kap * 2.0 ** -53 * np.linalg.norm(a)


@pytest.mark.parametrize("name,fmt", [("cfg1", "fp16"), ("cfg2w", "bf16"), ("cfg2w", "fp16")])
def test_explicit_inverse_same_solve(name, fmt):
    """The solve through W: the same status, RQI and PCG counts as substitution, and the
    SVD's x and sigma."""
    P = tlsgen.config(name)
    ex = exact.tls_svd(P.A, P.b)
    pc = rqi.factor_precond(P.A, fmt)
    r1 = rqi.rqi_pcgtls_mp(P.A, P.b, pc)
    r2 = rqi.rqi_pcgtls_mp(P.A, P.b, pc, opts=rqi.RqiOptions(precond_apply=2))
    assert (r2.status, r2.termination, r2.rqi_iters, r2.pcg_iters) == (r1.status, r1.termination, r1.rqi_iters, r1.pcg_iters)
    assert abs(r2.boot_iters - r1.boot_iters) <= 1
    assert np.linalg.norm(r2.x - ex.x) / np.linalg.norm(ex.x) <= 1e-12
    assert abs(r2.sigma - ex.sigma) / ex.sigma <= 1e-12


# ----------------------------------------------------------------------------- certificate
def test_dot2_against_exact_rationals():
    """dot2_rows (Dot2): within one rounding of the exact rational dot product (plus the
    Dot2 bound's u^2 cond term), on sums with heavy cancellation where plain fp64 fails."""
    from fractions import Fraction
    rng = np.random.default_rng(21)
    k = 40
    a = rng.standard_normal((8, k)) * 10.0 ** rng.integers(-8, 8, (8, k))
    b = rng.standard_normal((8, k))
    a[:, -1] = -(a[:, :-1] * b[:, :-1]).sum(axis=1) / b[:, -1]      # near-cancellation
    got = rqi.dot2_rows(a, b)
    for i in range(8):
        ex = sum(Fraction(float(a[i, j])) * Fraction(float(b[i, j])) for j in range(k))
        absd = sum(abs(Fraction(float(a[i, j])) * Fraction(float(b[i, j]))) for j in range(k))
        err = abs(Fraction(float(got[i])) - ex)
        assert err <= Fraction(2.0 ** -53) * abs(ex) + Fraction(4 * k * k) * Fraction(2.0 ** -106) * absd


def test_certify_sigma_exact_on_consistent_pair():
    """certify_sigma on the SPEC.md:213 2x2 TLS closed form (sigma^2 = 3 - sqrt(5),
    x = (sqrt(5) - 1)/2) and on a consistent system (sigma = 0 at x_true)."""
    A = np.array([[2.0], [0.0]])          # tests/golden/tls_2x2.txt
    b = np.array([1.0, 1.0])
    x = np.array([(math.sqrt(5.0) - 1.0) / 2.0])
    s = rqi.certify_sigma(A, b, x)
    assert s * s == pytest.approx(3.0 - math.sqrt(5.0), rel=1e-14)
    P = tlsgen.paper_problem("bjorck", eps=0.0)
    assert rqi.certify_sigma(P.A, P.b, P.x_true) < 1e-15


# ----------------------------------------------------------------------------- R28 certificate
def test_certificate_rhs_is_the_counter_based_vector():
    """r_j = ((j + 1) * 0x9E3779B97F4A7C15 mod 2^64 >> 11) 2^-53 - 1/2, recomputed with Python
    integers and exact rationals (the GPU generates the same bits, k_cert_rhs)."""
    from fractions import Fraction
    r = rqi.certificate_rhs(300)
    for j in range(300):
        h = ((j + 1) * 0x9E3779B97F4A7C15) % (1 << 64)
        assert Fraction(r[j]) == Fraction(h >> 11, 1 << 53) - Fraction(1, 2)


@pytest.mark.parametrize("u_f", ["fp16", "fp64"])
def test_minimality_certificate_against_closed_form(u_f):
    """A = U diag(s) V^T with s_n = 1e-2 known by construction: A^T A - sigma^2 I is positive
    definite iff sigma < s_n.  The certificate must accept sigma = 0.9 s_n
    and 0.5 s_n and reject sigma = 1.1 s_n, between s_n and s_{n-1}, and above s_1."""
    P = tlsgen.dense_problem(600, 30, 1e2, 1e-3, 12, twin=True)
    s = np.linalg.svd(P.A, compute_uv=False)
    pc = rqi.factor_precond(P.A, u_f)
    for sig, want in [(0.5 * s[-1], False), (0.9 * s[-1], False), (1.1 * s[-1], True),
                      (0.5 * (s[-1] + s[-2]), True), (2.0 * s[0], True)]:
        nm, dmin = rqi.minimality_certificate(P.A, pc, sig * sig, 10)
        assert nm == want, (sig / s[-1], dmin)


def test_not_minimal_reported_for_a_converged_non_minimal_pair():
    """A nearly non-generic problem (literal noise 1e-1 at kappa 1e2: sigma_{n+1} ~ sigma'_n)
    with the paper's breakdown rule and an until-tol budget: RQI converges (tol crossing) to a
    singular pair of [A, b] ABOVE sigma'_n -- an eigenpair, not the TLS solution.  With
    minimal_check the status is NOT_MINIMAL, and the SVD confirms sigma > sigma'_n; the same
    options on well-posed problems (cfg1, cfg2w) keep OK with sigma < sigma'_n."""
    P = tlsgen.dense_problem(400, 40, 1e2, 1e-1, 2, twin=False)
    sn = np.linalg.svd(P.A, compute_uv=False)[-1]
    o = rqi.RqiOptions(breakdown_rule=1, budget_rule=1, minimal_check=10)
    _, res = rqi.solve(P.A, P.b, "fp64", opts=o)
    assert res.status == rqi.NOT_MINIMAL and res.termination == rqi.T_CONVERGED_TOL
    assert res.sigma > sn
    _, res0 = rqi.solve(P.A, P.b, "fp64", opts=rqi.RqiOptions(breakdown_rule=1, budget_rule=1))
    assert res0.status == rqi.OK and res0.sigma == res.sigma          # the check changes only the status
    for name in ("cfg1", "cfg2w"):
        Q = tlsgen.config(name)
        _, r = rqi.solve(Q.A, Q.b, Q.u_f, opts=rqi.RqiOptions(minimal_check=10))
        assert r.status == rqi.OK and r.sigma < np.linalg.svd(Q.A, compute_uv=False)[-1]


# ----------------------------------------------------------------------------- stop rule (R6, R7)
@pytest.mark.parametrize("psis,opts,want", [
    # no crossing, psi rises at k = 3: STAGNATED with x_2 (R7)
    ([5.0, 4.0, 6.0], {}, (rqi.STAGNATED, rqi.T_STAGNATED, 3, 2)),
    # crossing at k = 2, polish step k = 3 improves: CONVERGED_TOL with x_3 (R6)
    ([5.0, 1e-20, 0.5e-20], {}, (rqi.OK, rqi.T_CONVERGED_TOL, 3, 3)),
    # crossing at k = 2, the polish step's psi rose: CONVERGED_TOL, the better iterate x_2 (R6)
    ([5.0, 1e-20, 2e-20], {}, (rqi.OK, rqi.T_CONVERGED_TOL, 3, 2)),
    # polish = 2: psi rises at k = 3 after the crossing at k = 2: PSI_INCREASE_CONVERGED with x_2
    ([5.0, 1e-20, 3e-20], {"polish": 2}, (rqi.OK, rqi.T_PSI_INCREASE_CONVERGED, 3, 2)),
    # the weak rule (l.532): an equal psi counts as an increase
    ([5.0, 4.0, 4.0], {"stop_rule": 1}, (rqi.STAGNATED, rqi.T_STAGNATED, 3, 2)),
    ([5.0, 4.0, 4.0, 3.0, 2.0], {"max_outer": 4}, (rqi.MAX_OUTER, rqi.T_MAX_OUTER, 5, 5)),
])
def test_stop_rule_branches_on_scripted_psi(monkeypatch, psis, opts, want):
    """The stop tests of rqi_pcgtls_mp (R6: tol crossing + polish; R7: psi increase before the
    crossing is STAGNATED; l.265 strict / l.532 weak; max_outer) on a scripted psi_k sequence:
    newton_residual is replaced by a script (sigma_k^2 = k, f = 0, g = 0, psi_k given) and each
    PCGTLS solve returns omega = e_0, so x_k = (k - 1) e_0 marks which iterate is returned."""
    n = 3
    A = np.eye(6, n)
    b = np.ones(6)
    pc = rqi.Precond(np.eye(n), np.ones(n), "fp64", 1.0)
    calls = {"k": 0}

    def script(A_, b_, x):
        k = calls["k"]
        calls["k"] += 1
        return float(k + 1), np.zeros(n), 0.0, psis[min(k, len(psis) - 1)]

    def pcg(A_, pc_, sigma2, f, l, tol_inner, variant="A", breakdown_rule="spec", A32=None):
        om = np.zeros(n)
        if sigma2 > 0:                                   # RQI solves (the bootstrap runs at sigma^2 = 0)
            om[0] = 1.0
        return rqi.PcgResult(om, l)

    monkeypatch.setattr(rqi, "newton_residual", script)
    monkeypatch.setattr(rqi, "pcgtls", pcg)
    o = rqi.RqiOptions(**opts)
    res = rqi.rqi_pcgtls_mp(A, b, pc, tol=1e-14, opts=o)
    status, term, k, k_ret = want
    assert (res.status, res.termination, res.rqi_iters) == (status, term, k)
    assert res.x[0] == k_ret - 1                        # x_{k_ret}
    assert res.sigma == pytest.approx(np.sqrt(k_ret))    # sigma_{k_ret}
