"""Pins of oracle/qr.py (Householder QR in u_q; SURVEY §8(f) NEXT-2 groundwork):
SPEC.md's worked examples, LAPACK agreement in fp64, the Gram residual bound in low
precision, and the paper's point that QR depends on kappa where the Gram Cholesky
depends on kappa^2."""
import math
from fractions import Fraction

import numpy as np
import pytest

from oracle.qr import householder_qr_r
from oracle.rounding import FORMATS, round_to, unit_roundoff


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
    """SPEC.md invariant 'QR residual <= 10 m n u' in Gram form (Q is not formed), with the
    probabilistic dimension factor of PAPER.md l.279-283 (sqrt(m) n^{3/4} instead of m n^{3/2}):
    ||R^T R - Ah^T Ah||_F <= c sqrt(m) n^{3/4} u ||Ah||_F^2, c = 2, Ah = fl(A).  At 60 x 12 the
    right side is 0.25 ||Ah||^2 in fp16 (2.0 in bf16, where only the exact rounding-point pin
    below binds), so R = 0 (residual = ||Ah^T Ah|| >= ||Ah||^2 / sqrt(n)) fails it in fp16/fp32."""
    rng = np.random.default_rng(5)
    m, n = 60, 12
    A = round_to(rng.standard_normal((m, n)), fmt)
    R = householder_qr_r(A, fmt)
    u = unit_roundoff(fmt)
    bound = 2 * np.sqrt(m) * n ** 0.75 * u * np.linalg.norm(A) ** 2
    assert np.linalg.norm(R.T @ R - A.T @ A) <= bound
    if fmt != "bf16":
        assert np.linalg.norm(A.T @ A) > bound          # the bound is not vacuous: R = 0 fails


# ---------------------------------------------------------------- exact rounding-point pin
def _rd_frac(x: Fraction, fmt: str) -> Fraction:
    """Round a rational to the nearest fmt value, ties to even (no floating point involved):
    the exact counterpart of oracle.rounding.round_to for finite, in-range values."""
    p, emin, _ = FORMATS[fmt]
    if x == 0:
        return Fraction(0)
    a = abs(x)
    e = a.numerator.bit_length() - a.denominator.bit_length()     # 2^e <= a < 2^(e+2)
    while Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    q = Fraction(2) ** (max(e, emin) - (p - 1))
    k, r = divmod(a / q, 1)
    k = int(k)
    if r > Fraction(1, 2) or (r == Fraction(1, 2) and k % 2 == 1):
        k += 1
    return (k * q) if x > 0 else -(k * q)


def _rd_sqrt_frac(y: Fraction, fmt: str) -> Fraction:
    """fmt value nearest to sqrt(y) (ties to even), decided by exact comparisons of squares."""
    p, emin, _ = FORMATS[fmt]
    s = _rd_frac(Fraction(math.sqrt(float(y))), fmt)            # a candidate within an ulp
    for _ in range(4):                                             # walk to the nearest one
        e = math.frexp(float(s))[1] - 1
        q = Fraction(2) ** (max(e, emin) - (p - 1))
        lo, hi = s - q / 2, s + q / 2                              # its rounding interval
        if hi * hi < y:
            s += q
        elif lo >= 0 and lo * lo > y:
            s -= q
        else:
            break
    return s


def _householder_qr_r_exact(A, fmt):
    """The R25 rounding points computed in exact rational arithmetic: every inner product is
    the EXACT sum rounded once to fmt, every elementwise step rounded once, sqrt correctly
    rounded.  Independent of oracle.qr (no numpy arithmetic, no float sums)."""
    rd = lambda x: _rd_frac(Fraction(x), fmt)
    m, n = len(A), len(A[0])
    W = [[rd(Fraction(float(A[i][j]))) for j in range(n)] for i in range(m)]
    for j in range(n):
        x = [W[i][j] for i in range(j, m)]
        sigma = _rd_sqrt_frac(rd(sum(t * t for t in x)), fmt)
        alpha = -sigma if x[0] >= 0 else sigma
        v = list(x)
        v[0] = rd(x[0] - alpha)
        beta = rd(Fraction(2) / rd(sum(t * t for t in v)))
        for k in range(j + 1, n):
            wk = rd(beta * rd(sum(v[i - j] * W[i][k] for i in range(j, m))))
            for i in range(j, m):
                W[i][k] = rd(W[i][k] - rd(v[i - j] * wk))
        W[j][j] = alpha
        for i in range(j + 1, m):
            W[i][j] = Fraction(0)
    R = [[W[i][k] if k >= i else Fraction(0) for k in range(n)] for i in range(n)]
    return [[(-e if R[i][i] < 0 else e) for e in R[i]] for i in range(n)]


@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
@pytest.mark.parametrize("shape,seed", [((4, 3), 0), ((4, 3), 1), ((4, 3), 2), ((5, 3), 3), ((4, 2), 4)])
def test_householder_rounding_points_exact(fmt, shape, seed):
    """householder_qr_r in fp16 / bf16 equals, bit for bit, the same rounding sequence done in
    exact rational arithmetic (fractions.Fraction): sigma, v_0, beta, every w_k and every
    updated entry rounded once to u_f at the points R25 names.  On these small inputs the
    oracle's fp64 inner products are exact, so any difference is a wrong rounding point (a
    missing or extra rounding, a rounded square before the sqrt, a wrong sign of alpha, an
    unrounded product) -- not a summation-order effect."""
    rng = np.random.default_rng(100 + seed)
    A = rng.standard_normal(shape) * np.array([1.0, 7.0, 0.3][: shape[1]])
    R = householder_qr_r(A, fmt)
    Rx = _householder_qr_r_exact(A.tolist(), fmt)
    assert np.array_equal(R, np.array([[float(e) for e in row] for row in Rx]))
    # and the exact sequence really differs from a no-rounding QR (the pin is not vacuous)
    R64 = householder_qr_r(A, "fp64")
    assert not np.array_equal(R, R64)


def test_exact_rounding_helpers():
    """The rational rounding agrees with oracle.rounding.round_to on ties, subnormals and
    random values, and the rational sqrt rounding is the nearest fp16 value."""
    rng = np.random.default_rng(9)
    for fmt in ("fp16", "bf16"):
        p, emin, _ = FORMATS[fmt]
        xs = list(rng.standard_normal(200) * 10.0 ** rng.uniform(-6, 3, 200))
        q = 2.0 ** (emin - (p - 1))
        xs += [q * 0.5, q * 1.5, q * 2.5, 1 + 2.0 ** -p, 1 + 3 * 2.0 ** -p]
        for x in xs:
            assert float(_rd_frac(Fraction(x), fmt)) == float(round_to(np.array([x]), fmt)[0])
        for y in rng.uniform(0.01, 100, 100):
            s = float(_rd_sqrt_frac(Fraction(y), fmt))
            cand = round_to(np.array([math.sqrt(y)]), fmt)[0]
            # nearest: no representable neighbour is closer to sqrt(y)
            nb = [np.nextafter(np.float16(cand), np.float16(np.inf)), np.nextafter(np.float16(cand), np.float16(-np.inf))] \
                if fmt == "fp16" else []
            assert abs(s - math.sqrt(y)) <= min([abs(float(t) - math.sqrt(y)) for t in nb] + [abs(s - math.sqrt(y))])
            assert s == cand


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
    """Two levels of Householder QR in fmt: ||R^T R - Ah^T Ah||_F <= 2 x (the one-level
    probabilistic Gram bound of test_gram_residual_bound, c = 2), and the leaf rounding
    points are the exact ones (each leaf R is householder_qr_r of its block, pinned by
    test_householder_rounding_points_exact; the stack is its own QR).  The bound is not vacuous
    in fp16 / fp32: R = 0 fails it."""
    from oracle.qr import even_row_blocks, tsqr_r
    rng = np.random.default_rng(5)
    m, n = 300, 12
    A = round_to(rng.standard_normal((m, n)) * np.logspace(0, -1, n)[None, :], fmt)
    bl = even_row_blocks(m, 3)
    R = tsqr_r(A, bl, fmt)
    u = unit_roundoff(fmt)
    assert np.all(np.diag(R) > 0)
    bound = 2 * 2 * np.sqrt(m) * n ** 0.75 * u * np.linalg.norm(A) ** 2
    assert np.linalg.norm(R.T @ R - A.T @ A) <= bound
    if fmt != "bf16":
        assert np.linalg.norm(A.T @ A) > bound
    # the stack is exactly the interleaved leaf R's
    Rs = [householder_qr_r(A[r0:r1], fmt, leaf=True) for r0, r1 in bl]
    S = np.zeros((3 * n, n))
    for b, Rb in enumerate(Rs):
        S[b::3] = Rb
    assert np.array_equal(R, householder_qr_r(S, fmt))


def test_tsqr_leaf_with_vanishing_column():
    """A full-rank A whose column 2 is zero on the first leaf's rows (a vanishing
    leaf column is not a rank deficiency).  The leaf takes the identity reflector (R_22 = 0),
    the stack factorization recovers A's R: in fp64 it equals LAPACK's R of A up to row signs;
    in fp16 the TSQR succeeds (no ZeroColumn) with a positive diagonal.  A column that is zero
    on ALL rows still raises from the stack."""
    from oracle.qr import ZeroColumn, even_row_blocks, tsqr_r
    rng = np.random.default_rng(21)
    A = rng.standard_normal((90, 6))
    A[:30, 2] = 0.0
    with pytest.raises(ZeroColumn):
        householder_qr_r(A[:30], "fp64")                   # the plain QR of the leaf raises
    R = tsqr_r(A, even_row_blocks(90, 3), "fp64")
    R0 = np.linalg.qr(A, mode="r")
    R0 = R0 * np.where(np.diag(R0) < 0, -1.0, 1.0)[:, None]
    assert np.max(np.abs(R - R0)) <= 1e-13 * np.max(np.abs(R0))
    R16 = tsqr_r(A, even_row_blocks(90, 3), "fp16")
    assert np.all(np.diag(R16) > 0)
    A[:, 2] = 0.0
    with pytest.raises(ZeroColumn) as e:
        tsqr_r(A, even_row_blocks(90, 3), "fp16")
    assert e.value.col == 2


def test_norm_scaling_is_the_papers_D_rounded():
    """R27: d_j is the power of two nearest to sqrt(c_j) = ||a_j||, checked by
    brute force over exponents in extended precision (math.log2 of an exactly representable
    c_j away from the boundaries c = 2^(2t+1)), and exactly at the boundaries: c = 2^(2t+1) ->
    sqrt(c) = 2^(t+1/2) rounds up to 2^(t+1) (ceil); c just below -> 2^t."""
    from oracle.rqi import norm_scaling
    rng = np.random.default_rng(8)
    A = rng.standard_normal((50, 40)) * 10.0 ** rng.uniform(-8, 8, 40)[None, :]
    d, nrm2 = norm_scaling(A)
    c = np.sum(A * A, axis=0)
    assert nrm2 == pytest.approx(np.sum(c), rel=1e-14)
    for cj, dj in zip(c, d):
        best = min(range(-40, 40), key=lambda t: abs(0.5 * math.log2(cj) - t))
        assert dj == 2.0 ** best
        assert 0.5 <= cj / dj ** 2 < 2.0
    for t in (-3, 0, 5):
        B = np.zeros((2, 2))
        B[0, 0] = math.sqrt(2.0 ** (2 * t + 1))      # c = 2^(2t+1) up to one rounding of the sqrt
        B[:, 1] = [2.0 ** t, 2.0 ** t]                # c = 2^(2t+1) exactly
        d2, _ = norm_scaling(B)
        assert d2[1] == 2.0 ** (t + 1)


# ---------------------------------------------------------------- blocked QR (R29, NEXT-2)
def test_blocked_fp64_equals_lapack_and_b_ge_n_is_unblocked():
    """R29's compact-WY trailing update is the unblocked factorization in exact arithmetic: in
    fp64 it gives LAPACK's R (up to row signs) for panel widths that divide n and that do not,
    and with b >= n it is householder_qr_r bit for bit (no trailing update happens)."""
    from oracle.qr import householder_qr_r_blocked
    rng = np.random.default_rng(31)
    A = rng.standard_normal((120, 21))
    R0 = np.linalg.qr(A, mode="r")
    R0 = R0 * np.where(np.diag(R0) < 0, -1.0, 1.0)[:, None]
    for b in (2, 5, 7, 16):
        assert np.max(np.abs(householder_qr_r_blocked(A, "fp64", b) - R0)) <= 1e-13 * np.max(np.abs(R0))
    for fmt in ("fp16", "bf16"):
        assert np.array_equal(householder_qr_r_blocked(A, fmt, 21), householder_qr_r(A, fmt))
        assert np.array_equal(householder_qr_r_blocked(A, fmt, 64), householder_qr_r(A, fmt))


def _blocked_exact(A, fmt, b):
    """R29 in exact rational arithmetic: the panel steps as _householder_qr_r_exact, the fp32
    chunk sums and the fp32 V Y sums rounded to fp32 (exact RNE of rationals) term by term."""
    rd = lambda x: _rd_frac(Fraction(x), fmt)
    r32 = lambda x: _rd_frac(Fraction(x), "fp32")
    m, n = len(A), len(A[0])
    W = [[rd(Fraction(float(A[i][j]))) for j in range(n)] for i in range(m)]
    for c0 in range(0, n, b):
        c1 = min(n, c0 + b)
        nb = c1 - c0
        V = [[Fraction(0)] * nb for _ in range(m - c0)]
        beta = [Fraction(0)] * nb
        for j in range(c0, c1):
            x = [W[i][j] for i in range(j, m)]
            sigma = _rd_sqrt_frac(rd(sum(t * t for t in x)), fmt)
            alpha = -sigma if x[0] >= 0 else sigma
            v = list(x)
            v[0] = rd(x[0] - alpha)
            bt = rd(Fraction(2) / rd(sum(t * t for t in v)))
            for k in range(j + 1, c1):
                wk = rd(bt * rd(sum(v[i - j] * W[i][k] for i in range(j, m))))
                for i in range(j, m):
                    W[i][k] = rd(W[i][k] - rd(v[i - j] * wk))
            W[j][j] = alpha
            for i in range(j + 1, m):
                W[i][j] = Fraction(0)
            for i in range(j, m):
                V[i - c0][j - c0] = v[i - j]
            beta[j - c0] = bt
        if c1 == n:
            break
        def chunk_dot(a_col, b_col):              # fp32 row-order sums per 64-row chunk, fp64 across
            tot = Fraction(0)
            for s0 in range(0, m - c0, 64):
                acc = Fraction(0)
                for i in range(s0, min(m - c0, s0 + 64)):
                    acc = r32(acc + a_col(i) * b_col(i))
                tot = tot + acc                   # fp64 sums of a few fp32 values: exact here
            return tot
        VtC = [[chunk_dot(lambda i: V[i][p], lambda i: W[c0 + i][k]) for k in range(c1, n)] for p in range(nb)]
        VtV = [[chunk_dot(lambda i: V[i][p], lambda i: V[i][q]) for q in range(nb)] for p in range(nb)]
        T = [[Fraction(0)] * nb for _ in range(nb)]
        for j in range(nb):
            T[j][j] = beta[j]
            for i in range(j):
                T[i][j] = -beta[j] * sum(T[i][l] * VtV[l][j] for l in range(j))
        Y = [[rd(sum(T[l][p] * VtC[l][k] for l in range(nb))) for k in range(n - c1)] for p in range(nb)]
        for i in range(m - c0):
            for k in range(n - c1):
                acc = Fraction(0)
                for p in range(nb):
                    acc = r32(acc + V[i][p] * Y[p][k])
                W[c0 + i][c1 + k] = rd(W[c0 + i][c1 + k] - acc)
    R = [[W[i][k] if k >= i else Fraction(0) for k in range(n)] for i in range(n)]
    return [[(-e if R[i][i] < 0 else e) for e in R[i]] for i in range(n)]


@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
@pytest.mark.parametrize("shape,b,seed", [((8, 5), 2, 0), ((9, 6), 3, 1), ((7, 4), 1, 2)])
def test_blocked_rounding_points_exact(fmt, shape, b, seed):
    """householder_qr_r_blocked equals R29's rounding sequence evaluated in exact rational
    arithmetic.  The fp64 pieces (T, T^T V^T C before its single rounding) are exact in
    rationals and within fp64 rounding in the oracle; on these inputs that never moves a u_f
    result, and every u_f / fp32 rounding point must match."""
    from oracle.qr import householder_qr_r_blocked
    rng = np.random.default_rng(200 + seed)
    A = rng.standard_normal(shape) * np.array([1.0, 3.0, 0.5, 2.0, 0.7, 1.3][: shape[1]])
    R = householder_qr_r_blocked(A, fmt, b)
    Rx = _blocked_exact(A.tolist(), fmt, b)
    assert np.array_equal(R, np.array([[float(e) for e in row] for row in Rx]))
    assert not np.array_equal(R, householder_qr_r_blocked(A, "fp64", b))


@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
def test_blocked_backward_error_and_preconditioner(fmt):
    """The blocked fp16 / bf16 R~ satisfies the same probabilistic Gram residual bound as the
    unblocked one (R = 0 fails it in fp16), stays within a few u_f of it, and preconditions A
    as well: kappa(A R~^{-1}) < 10 at kappa(A) = 300."""
    from oracle.qr import householder_qr_r_blocked
    rng = np.random.default_rng(41)
    m, n = 400, 24
    U, _ = np.linalg.qr(rng.standard_normal((m, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)))
    A = (U * np.logspace(0, -np.log10(300.0), n)) @ V.T
    Ah = round_to(A, fmt)
    Rb = householder_qr_r_blocked(A, fmt, 8)
    Ru = householder_qr_r(A, fmt)
    u = unit_roundoff(fmt)
    bound = 2 * np.sqrt(m) * n ** 0.75 * u * np.linalg.norm(Ah) ** 2
    assert np.linalg.norm(Rb.T @ Rb - Ah.T @ Ah) <= bound
    if fmt == "fp16":
        assert np.linalg.norm(Ah.T @ Ah) > bound
    assert np.linalg.norm(Rb - Ru) <= 50 * u * np.linalg.cond(Ah) * np.linalg.norm(Ru)
    assert np.linalg.cond(A @ np.linalg.inv(Rb)) < 10.0
