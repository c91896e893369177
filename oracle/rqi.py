"""Algorithmic oracle: RQI-PCGTLS-MP on the CPU in fp64 with emulated u_f
rounding (oracle c2; TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

Follows, in the paper's order and notation:
  Alg. 4 RQI-PCGTLS-MP    PAPER.md l.221-258 (§3)
  Alg. 3 l-step PCGTLS    PAPER.md l.186-204 (§2), operator of l.322-328 (§3.1)
  psi_k termination       PAPER.md l.260-265 (Eq. psik)
  scaled Cholesky         PAPER.md l.290-307 (§3.1)
Where the paper is silent or ambiguous the DESIGN.md reading is cited as R<n>.

The u_f rounding is applied exactly where the GPU path rounds (R10): the scaled
matrix A D^{-1} before the Gram, the Gram's fp32 accumulation per chunk of K_t
rows (fp16/bf16 only), and the Cholesky factor R -> R~ = fl_uf(R).  Everything
else is fp64 (u = u_r = fp64, BASELINE north_star).

A may be a dense numpy array or a scipy.sparse CSR matrix (BASELINE cfg3).
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import numpy as np
import scipy.linalg
import scipy.linalg.lapack
import scipy.sparse

from .rounding import round_to

# status codes (include/tlsrqi.h mirrors the numbers; the oracle does not read it)
OK, CHOL_BREAKDOWN, PCG_BREAKDOWN, MAX_OUTER, NONFINITE, RANGE, NOT_MINIMAL, STAGNATED = range(8)
# termination reasons
T_NONE, T_CONVERGED_TOL, T_PSI_INCREASE_CONVERGED, T_STAGNATED, T_MAX_OUTER, T_BREAKDOWN, T_NONFINITE = range(7)


# ----------------------------------------------------------------------------- helpers
def _is_sparse(A) -> bool:
    return scipy.sparse.issparse(A)


def matvec(A, x):
    return np.asarray(A @ x).reshape(-1)


def rmatvec(A, t):
    return np.asarray(A.T @ t).reshape(-1)


# ----------------------------------------------------------------------------- scaling
def column_scaling(A):
    """Exact two-sided scaling stand-in (reading R2):
    d_j = 2^floor(log2 max_i |a_ij|), so that |a_ij / d_j| < 2 and the scaling
    itself is exact (the paper assumes it "without incurring additional
    rounding error", l.307).  Also returns ||A||_F^2 for the tol stop (R6).
    A zero column makes A rank deficient (PAPER.md l.30 rank(A) = n): ValueError."""
    if _is_sparse(A):
        amax = np.asarray(abs(A).max(axis=0).todense()).reshape(-1)
        normA2 = float(A.multiply(A).sum())
    else:
        amax, c = _col_max_sumsq(np.asarray(A))
        normA2 = float(np.sum(c))
    if np.any(amax == 0) or not np.all(np.isfinite(amax)):
        raise ValueError("A has a zero or non-finite column")
    _, E = np.frexp(amax)
    d = np.ldexp(1.0, E - 1)
    return d, normA2


def _col_max_sumsq(A: np.ndarray):
    """Column maxima of |A| and column sums of squares, over row slices in the thread pool
    (the maxima are exact in any order; the sums of squares are fp64 sums of the row
    slices' sums, added in slice order)."""
    step = max(1, min(65536, -(-A.shape[0] // _threads())))
    sls = [slice(i, i + step) for i in range(0, A.shape[0], step)]
    def one(sl):
        X = A[sl]
        return np.max(np.abs(X), axis=0), np.einsum("ij,ij->j", X, X)
    parts = list(_pool().map(one, sls))
    amax = np.max(np.stack([p[0] for p in parts]), axis=0)
    c = np.zeros(A.shape[1])
    for p in parts:
        c += p[1]
    return amax, c


def norm_scaling(A):
    """The scaling of the QR route (reading R27): the paper's D, "a diagonal matrix with the
    square root of the diagonal elements of A^T A on the diagonal", rounded
    to a power of two so that applying it is exact (l.307): with c_j = ||a_j||^2 and
    k = floor(log2 c_j), d_j = 2^ceil(k/2) is sqrt(c_j) rounded to the nearest power of two
    (sqrt(c_j) lies in [2^(k/2), 2^((k+1)/2))), and every scaled column has
    ||a_j/d_j||^2 in [1/2, 2).  Decided on powers of two of c_j, never on a rounded sqrt.
    Returns (d, ||A||_F^2); a zero or non-finite column raises ValueError (rank deficient)."""
    if _is_sparse(A):
        c = np.asarray(A.multiply(A).sum(axis=0)).reshape(-1)
    else:
        c = _col_max_sumsq(np.asarray(A))[1]
    if np.any(c == 0) or not np.all(np.isfinite(c)):
        raise ValueError("A has a zero or non-finite column")
    _, E = np.frexp(c)                 # c = f 2^E, f in [1/2, 1): k = E - 1
    k = E - 1
    d = np.ldexp(1.0, -((-k) // 2))    # 2^ceil(k/2)
    return d, float(np.sum(c))


# ----------------------------------------------------------------------------- Gram
def _gram_sparse(A, d: np.ndarray, u_f: str) -> np.ndarray:
    """CSR A (reading R19): no tensor-core chunks on this path, so G = A^^T A^ with
    A^ = fl_uf(A D^{-1}) is the exact sum of the exact u_f products, rounded ONCE
    to fp64.  fp16: every A^ entry is an integer multiple of 2^-24 with |A^| < 2
    (column scaling R2), so I = A^ 2^24 is an integer below 2^25; I = H 2^13 + L
    (0 <= L < 2^13) keeps the three integer products H^T H, H^T L + L^T H, L^T L
    exact in int64, and their exact combination is rounded by Python's
    correctly rounded int -> float.  bf16/fp32/fp64: the products (exact for
    bf16/fp32) summed in fp64 by scipy."""
    A = scipy.sparse.csr_matrix(A)
    Ah = A.copy()
    Ah.data = round_to(A.data / d[A.indices], u_f)
    if not np.all(np.isfinite(Ah.data)):
        raise OverflowError("A D^-1 overflows u_f")
    if u_f != "fp16":
        return np.asarray((Ah.T @ Ah).todense())
    scaled = Ah.data * 2.0 ** 24
    I = scaled.astype(np.int64)
    assert np.array_equal(I.astype(np.float64), scaled)         # exact integers
    Hm, Lm = Ah.copy(), Ah.copy()
    Hm.data, Lm.data = I >> 13, I & 8191
    Hm = Hm.astype(np.int64)
    Lm = Lm.astype(np.int64)
    SA = np.asarray((Hm.T @ Hm).todense(), dtype=np.int64)
    SB = np.asarray((Hm.T @ Lm + Lm.T @ Hm).todense(), dtype=np.int64)
    SC = np.asarray((Lm.T @ Lm).todense(), dtype=np.int64)
    T = SA.astype(object) * (1 << 26) + SB.astype(object) * (1 << 13) + SC.astype(object)
    G = np.array([float(t) for t in T.ravel()], dtype=np.float64).reshape(T.shape)
    return G * 2.0 ** -48


def _round_rows(X: np.ndarray, d: np.ndarray, u_f: str, out_dtype) -> np.ndarray:
    """fl_uf(X D^{-1}) (round_to) computed on row slices in a thread pool (numpy releases
    the GIL), returned as out_dtype (exact: the values are u_f values); fp16 through
    numpy's float16 cast, which is the same direct fp64 -> fp16 RNE (pinned bit-exact
    against round_to in tests/test_oracle_rounding.py).  OverflowError if any value
    overflows u_f."""
    out = np.empty(X.shape, dtype=out_dtype)
    def one(sl):
        Y = X[sl] / d[None, :]
        if u_f == "fp16":
            with np.errstate(over="ignore"):
                Y = Y.astype(np.float16)
        else:
            Y = round_to(Y, u_f)
        out[sl] = Y
        return bool(np.all(np.isfinite(out[sl])))
    step = max(1, -(-X.shape[0] // _threads()))
    sls = [slice(i, i + step) for i in range(0, X.shape[0], step)]
    if not all(_pool().map(one, sls)):
        raise OverflowError("A D^-1 overflows u_f")
    return out


_POOL = None


def _threads() -> int:
    import os
    return max(1, min(32, os.cpu_count() or 1))


def _pool():
    global _POOL
    if _POOL is None:
        import concurrent.futures
        _POOL = concurrent.futures.ThreadPoolExecutor(_threads())
    return _POOL


def gram_uf(A, d: np.ndarray, u_f: str, K_t: int = 64) -> np.ndarray:
    """Dense A:  G = sum over chunks c of K_t consecutive rows (in order) of
    fp64( fl32-accumulated  A^_c^T A^_c ),  A^ = fl_uf(A D^{-1})   (R10, R11).

    u_f in {fp16, bf16}: the products of u_f values are exact in fp32 and each
    chunk is summed in fp32 (a float32 matmul), as the tensor cores accumulate
    in fp32; the chunk sums are added to G in fp64 in chunk order.  u_f = fp32:
    A^ in fp32, the chunk products formed in fp64.  u_f = fp64: G = (A D^{-1})^T
    (A D^{-1}) in fp64 (control).

    Evaluation (no change to the arithmetic above): rows are rounded in slices of
    64 chunks, the chunk products of a slice are one batched matmul, and the output
    rows are split over a thread pool; every element of G still receives its
    chunk sums one at a time in chunk order."""
    if _is_sparse(A):
        return _gram_sparse(A, d, u_f)
    m, n = A.shape
    G = np.zeros((n, n))
    low = u_f in ("fp16", "bf16")
    nb = max(1, min(_threads(), -(-n // 64)))
    rblocks = [slice(j * n // nb, (j + 1) * n // nb) for j in range(nb)]
    rows = K_t * 64
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):          # one BLAS thread per pool thread
        for r0 in range(0, m, rows):
            blk = A[r0:r0 + rows]
            blk = blk.toarray() if _is_sparse(blk) else np.asarray(blk)
            Ah = _round_rows(blk, d, u_f, np.float32 if low else np.float64)
            nfull = Ah.shape[0] // K_t
            chunks = [Ah[: nfull * K_t].reshape(nfull, K_t, n)] if nfull else []
            tail = Ah[nfull * K_t:]

            def work(rb):
                Gr = G[rb]                                        # rows rb of G (a view)
                for C in chunks:                                  # (nc, K_t, n)
                    S = np.matmul(C[:, :, rb].transpose(0, 2, 1), C)   # (nc, |rb|, n), fp32 or fp64
                    for c in range(S.shape[0]):                   # chunk order
                        Gr += S[c]
                if tail.shape[0]:
                    Gr += tail[:, rb].T @ tail

            list(_pool().map(work, rblocks))
    return G


def gram_exact_bound(A, d: np.ndarray, u_f: str, K_t: int = 64) -> np.ndarray:
    """Elementwise bound on |G_fp32chunks - A^^T A^| (standard dot-product error
    bound, gamma_k = k u/(1 - k u) with u = 2^-24 per fp32 chunk of length <= K_t,
    plus the fp64 chunk sums)."""
    m, n = A.shape
    B = np.zeros((n, n))
    u32 = 2.0 ** -24
    k = min(K_t, m)
    gam = k * u32 / (1 - k * u32)
    for c0 in range(0, m, K_t):
        blk = A[c0:c0 + K_t]
        blk = blk.toarray() if _is_sparse(blk) else np.asarray(blk)
        Ah = np.abs(round_to(blk / d[None, :], u_f))
        B += Ah.T @ Ah
    nchunks = (m + K_t - 1) // K_t
    return (gam + (nchunks + 1) * 2.0 ** -53) * B


def gram_accumulation_bound(A, d: np.ndarray, u_f: str, K_t: int = 64, super_chunks: int = 64,
                            truncating: bool = True, nsplit: int = 148) -> np.ndarray:
    """Elementwise bound on |G - A^^T A^| for every member of the accumulation family that
    reading R11 fixes for the dense u_f in {fp16, bf16} Gram:
      level 1  each K_t-row chunk summed in fp32 (the tensor cores): unit u1 = 2^-23 when the
               adder truncates (R11 measured a truncation bias), 2^-24 for round-to-nearest;
      level 2  `super_chunks` consecutive chunk sums added in fp32, round to nearest (2^-24);
      level 3  everything after that in fp64: the flushes of one row split and `nsplit` splits.
    With gamma(k, u) = k u / (1 - k u) and S = |A^|^T |A^| (the exact products are exact):
      |G - A^^T A^| <= [ (1 + g1)(1 + g2)(1 + g3) - 1 ] S,
      g1 = gamma(K_t - 1, u1),  g2 = gamma(super_chunks - 1, 2^-24),
      g3 = gamma(ceil(m / (K_t super_chunks)) + nsplit, 2^-53),
    the standard recursive-summation bound applied level by level (each level's inputs are the
    previous level's computed sums, whose magnitudes are bounded by (1 + g) times the exact
    sums of |products|).  gram_exact_bound is the one-level special case."""
    m = A.shape[0]
    def gam(k, u):
        k = max(int(k), 0)
        return k * u / (1.0 - k * u)
    g1 = gam(min(K_t, m) - 1, 2.0 ** -23 if truncating else 2.0 ** -24)
    g2 = gam(min(super_chunks, -(-m // K_t)) - 1, 2.0 ** -24)
    g3 = gam(-(-m // (K_t * super_chunks)) + nsplit, 2.0 ** -53)
    S = np.zeros((A.shape[1], A.shape[1]))
    for c0 in range(0, m, 65536):
        blk = A[c0:c0 + 65536]
        blk = blk.toarray() if _is_sparse(blk) else np.asarray(blk)
        Ah = np.abs(round_to(blk / d[None, :], u_f))
        S += Ah.T @ Ah
    return ((1 + g1) * (1 + g2) * (1 + g3) - 1) * S


# ----------------------------------------------------------------------------- Cholesky
@dataclasses.dataclass
class Precond:
    """P = R~ D with P^T P ~ A^T A."""
    Rt: np.ndarray      # R~ = fl_uf(R), n x n upper triangular, values held in fp64
    d: np.ndarray       # column scaling, powers of two
    u_f: str
    normA2: float       # ||A||_F^2
    status: int = OK
    chol_pivot: int = 0  # 1-based index of the first failed pivot (CHOL_BREAKDOWN)
    G: Optional[np.ndarray] = None
    R: Optional[np.ndarray] = None
    W: Optional[np.ndarray] = None   # explicit inverse of R~ when the solve applies it (R24)


def factor_precond_qr(A, u_f: str, row_blocks=None) -> Precond:
    """The paper's preferred preconditioner: R~ = the R factor
    of a Householder QR of A D^{-1} computed with every operation in u_f (oracle/qr.py,
    reading R25), scaled by the paper's D = diag(A^T A)^{1/2} rounded to powers of two
    (norm_scaling, reading R27; GPU: tls_factor_precond_qr).  row_blocks: the TSQR leaves (R26)."""
    from .qr import householder_qr_r, tsqr_r
    A_d = A.toarray() if _is_sparse(A) else np.asarray(A)
    n = A_d.shape[1]
    d, normA2 = norm_scaling(A)
    try:
        # row_blocks: the TSQR leaves of a row-sharded A (R26); None = one block
        Rt = householder_qr_r(A_d / d, u_f) if row_blocks is None else tsqr_r(A_d / d, row_blocks, u_f)
    except ZeroDivisionError as e:   # 1-based index of the vanishing column (tlsrqi.h chol_pivot)
        return Precond(np.zeros((n, n)), d, u_f, normA2, CHOL_BREAKDOWN, getattr(e, "col", 0) + 1)
    if not np.all(np.isfinite(Rt)) or np.any(np.diag(Rt) == 0):
        return Precond(Rt, d, u_f, normA2, RANGE)
    return Precond(Rt, d, u_f, normA2, OK)


def factor_precond(A, u_f: str, K_t: int = 64, keep: bool = False) -> Precond:
    """tls_factor_precond: scaling, u_f Gram, fp64 Cholesky G = R^T R (LAPACK
    dpotrf, upper), R~ = fl_uf(R)  (PAPER.md l.231 with the Cholesky route of
    l.290-307; readings R10, R11)."""
    n = A.shape[1]
    d, normA2 = column_scaling(A)
    try:
        G = gram_uf(A, d, u_f, K_t)
    except OverflowError:
        return Precond(np.zeros((n, n)), d, u_f, normA2, RANGE)
    R, info = scipy.linalg.lapack.dpotrf(G, lower=0, clean=1)
    if info > 0 or not np.all(np.isfinite(np.diag(R))):
        piv = int(info) if info > 0 else int(np.argmin(np.isfinite(np.diag(R)))) + 1
        return Precond(np.zeros((n, n)), d, u_f, normA2, CHOL_BREAKDOWN, piv,
                       G if keep else None)
    Rt = round_to(np.triu(R), u_f)
    if not np.all(np.isfinite(Rt)) or np.any(np.diag(Rt) == 0):
        return Precond(Rt, d, u_f, normA2, RANGE)
    return Precond(Rt, d, u_f, normA2, OK, 0, G if keep else None, R if keep else None)


def with_inverse(pc: Precond) -> Precond:
    """The same preconditioner applied through W = R~^{-1}, formed once in fp64 by
    triangular solves against the identity (reading R24: tls_rqi_opts_t.precond_apply = 2)."""
    W = scipy.linalg.solve_triangular(pc.Rt, np.eye(pc.Rt.shape[0]), lower=False)
    return dataclasses.replace(pc, W=np.triu(W))


def apply_Pinv(pc: Precond, y: np.ndarray) -> np.ndarray:
    """P^{-1} y = D^{-1} (R~^{-1} y): back substitution (Alg. 3 l.193;
    Table 1 "Forward/Backward Subs", l.427), or D^{-1} (W y) with the explicit inverse (R24)."""
    if pc.W is not None:
        return (pc.W @ y) / pc.d
    return scipy.linalg.solve_triangular(pc.Rt, y, lower=False) / pc.d


def apply_PinvT(pc: Precond, y: np.ndarray) -> np.ndarray:
    """P^{-T} y = R~^{-T} (D^{-1} y): forward substitution (Alg. 3 l.191, l.197), or
    W^T (D^{-1} y) with the explicit inverse (R24)."""
    if pc.W is not None:
        return pc.W.T @ (y / pc.d)
    return scipy.linalg.solve_triangular(pc.Rt, y / pc.d, trans="T", lower=False)


# ----------------------------------------------------------------------------- PCGTLS
@dataclasses.dataclass
class PcgResult:
    omega: np.ndarray
    count: int              # number of alpha-updates executed (R3)
    breakdown: bool = False
    breakdown_j: int = -1
    delta_min: float = math.inf


def operator_fp32(A32, q: np.ndarray):
    """The A-in-loop operator at u_p = fp32 (reading R23; PAPER.md l.480-482 run PCGTLS
    in single): q rounded to fp32 (RNE), t = A32 q and v = A32^T t each accumulated in
    fp32 (numpy's float32 matrix-vector products), t^T t in fp64 of the fp32 t.
    Returns (t^T t, v) in fp64."""
    q32 = q.astype(np.float32)
    t = np.asarray(A32 @ q32, dtype=np.float32).reshape(-1)
    t64 = t.astype(np.float64)
    v = np.asarray(A32.T @ t, dtype=np.float32).reshape(-1).astype(np.float64)
    return float(t64 @ t64), v


def pcgtls(A, pc: Precond, sigma2: float, f: np.ndarray, l: int, tol_inner: float,
           variant: str = "A", breakdown_rule: str = "spec", A32=None) -> PcgResult:
    """l-step PCGTLS for (A^T A - sigma^2 I) omega = f (Alg. 3, l.186-204).

    variant "A" (default, reading R1): the preconditioned operator
        C^ = P^{-T}(A^T A - sigma^2 I) P^{-1}
    applied with A in the loop: t = A q, delta = t^T t - sigma^2 q^T q,
    w = P^{-T}(A^T t - sigma^2 q).
    variant "paper": Alg. 3 as printed, C~ = I - sigma^2 P^{-T} P^{-1} (l.206):
    delta = p^T p - sigma^2 q^T q (l.194), w = p - sigma^2 P^{-T} q (l.197-198).
    Loop guard (R3): delta non-finite or zero stops before the update (l.192);
    delta < 0 is a breakdown under the "spec" rule; at most l updates (R3);
    early exit after an update when eta_{j+1} <= tol_inner^2 eta_0.
    A32 (variant "A" only): the fp32 copy of A; the operator then runs at u_p = fp32
    (operator_fp32, R23) and everything else stays fp64."""
    n = f.shape[0]
    omega = np.zeros(n)                        # l.191
    s = apply_PinvT(pc, f)
    p = s.copy()
    eta = float(s @ s)
    eta0 = eta
    res = PcgResult(omega, 0)
    if eta0 == 0.0:
        return res
    for j in range(l):                         # l.192
        q = apply_Pinv(pc, p)                  # l.193
        if variant == "A" and A32 is not None:
            tt, v = operator_fp32(A32, q)
            delta = tt - sigma2 * float(q @ q)
        elif variant == "A":
            t = matvec(A, q)
            delta = float(t @ t) - sigma2 * float(q @ q)
        else:
            delta = float(p @ p) - sigma2 * float(q @ q)   # l.194
        res.delta_min = min(res.delta_min, delta)
        if not math.isfinite(delta) or delta == 0.0:
            break
        if delta < 0.0 and breakdown_rule == "spec":
            res.breakdown, res.breakdown_j = True, j
            break
        alpha = eta / delta                    # l.195
        omega = omega + alpha * q              # l.196
        if variant == "A" and A32 is not None:
            w = apply_PinvT(pc, v - sigma2 * q)
        elif variant == "A":
            w = apply_PinvT(pc, rmatvec(A, t) - sigma2 * q)
        else:
            w = p - sigma2 * apply_PinvT(pc, q)            # l.197
        s = s - alpha * w                      # l.198
        eta_new = float(s @ s)                 # l.199
        res.count += 1
        if eta_new <= tol_inner * tol_inner * eta0:
            break
        beta = eta_new / eta                   # l.200
        p = s + beta * p                       # l.201
        eta = eta_new
    res.omega = omega
    return res


# ----------------------------------------------------------------------------- RQI
@dataclasses.dataclass
class RqiOptions:
    """Mirrors tls_rqi_opts_t (include/tlsrqi.h); defaults are DESIGN.md's."""
    budget_rule: int = 0       # 0: k+1 PCG steps at RQI step k; 1: until tol (cap 400)
    stop_rule: int = 0         # 0: strict psi increase (l.265); 1: weak (>=, l.532)
    max_outer: int = 50
    polish: int = 1            # RQI steps taken after the tol crossing (R6)
    tol_inner: float = -1.0    # <= 0 -> tol
    boot: int = 0              # 0: x_LS by preconditioned CGLS (R5); 1: semi-normal
    boot_tol: float = 1e-8
    boot_max: int = 200
    op_variant: int = 0        # 0: A-in-loop (R1); 1: paper Alg. 3
    breakdown_rule: int = 0    # 0: delta <= 0 stops (spec); 1: delta == 0 only (paper)
    gram_chunk: int = 64
    u_p: str = "fp64"          # operator precision of the RQI's inner solves (R23): "fp64" | "fp32"
    precond_apply: int = 0     # R24: 1 substitution, 2 explicit inverse, 0 auto (= 1 in this one-process oracle)
    minimal_check: int = 0     # R28: PCG steps of the minimality certificate after an OK solve (0 = off)


@dataclasses.dataclass
class RqiResult:
    x: np.ndarray
    sigma: float
    status: int
    termination: int
    rqi_iters: int
    boot_iters: int
    pcg_iters: List[tuple]
    sigma2_trace: List[float]
    psi_trace: List[float]
    breakdown_k: int = -1
    breakdown_rhs: int = -1
    breakdown_j: int = -1
    passes: int = 0            # passes over A (unbatched) for perf accounting
    delta_min_trace: List[tuple] = dataclasses.field(default_factory=list)   # c2 step 9


def certificate_rhs(n: int) -> np.ndarray:
    """The fixed right-hand side of the minimality certificate (R28), a counter-based
    pseudo-random vector both sides generate bit for bit: h_j = (j + 1) * 0x9E3779B97F4A7C15
    mod 2^64, r_j = (h_j >> 11) 2^-53 - 1/2 (every step exact in fp64)."""
    h = np.arange(1, n + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    return (h >> np.uint64(11)).astype(np.float64) * 2.0 ** -53 - 0.5


def minimality_certificate(A, pc: Precond, sigma2: float, steps: int):
    """Is A^T A - sigma^2 I positive definite (x_TLS is unique only if
    sigma'_n > sigma_{n+1}, and PCGTLS needs A^T A - sigma_k^2 I SPD)?  Reading R28: `steps`
    iterations of PCGTLS (A-in-loop, l.186-204) at sigma^2 on certificate_rhs with no early
    exit.  CG's curvatures delta_j = p_j^T C p_j of C = P^{-T}(A^T A - sigma^2 I)P^{-1} are the
    pivots of the Lanczos tridiagonal T_j, so all delta_j > 0 <=> T_j SPD <=> every Ritz value
    of C is positive; a delta_j <= 0 exhibits a direction of non-positive curvature, so C -- and
    by Sylvester's law of inertia A^T A - sigma^2 I -- is not positive definite: sigma >= sigma'_n
    and (x, sigma) is not the TLS solution (NOT_MINIMAL).  The converse is one-sided: `steps`
    positive pivots make negative curvature unlikely (Lanczos finds extreme eigenvalues first),
    not impossible.  Returns (not_minimal, delta_min)."""
    n = A.shape[1]
    r = pcgtls(A, pc, sigma2, certificate_rhs(n), steps, 0.0, "A", "spec")
    return bool(r.breakdown or r.delta_min <= 0.0), r.delta_min


def newton_residual(A, b: np.ndarray, x: np.ndarray):
    """One outer residual evaluation (Alg. 4 l.238-245 and Eq. psik l.262):
    r = b - A x, sigma^2 = r^T r/(1 + x^T x), f = -A^T r - sigma^2 x (x read as x_k,
    reading R15), g = -b^T r + sigma^2, psi = ((f^T f + g^2)/(x^T x + 1))^{1/2}."""
    r = b - matvec(A, x)                   # l.238
    v = rmatvec(A, r)
    xx = float(x @ x)
    sig2 = float(r @ r) / (1.0 + xx)       # l.240
    f = -v - sig2 * x                      # l.242
    g = -float(b @ r) + sig2               # l.244
    psi = math.sqrt((float(f @ f) + g * g) / (xx + 1.0))   # l.262
    return sig2, f, g, psi


def rqi_pcgtls_mp(A, b: np.ndarray, pc: Precond, tol: float = 1e-14,
                  opts: Optional[RqiOptions] = None) -> RqiResult:
    """RQI-PCGTLS-MP, Alg. 4 (l.221-258), u = u_r = fp64 and the
    preconditioner R~ stored in u_f.  Stop tests (R6), in this order at step k
    after the residual pass:
      (ii) k* = first k with psi_k <= tol ||[A,b]||_F^2; at k = k* + polish
           return CONVERGED_TOL with (x_k, sigma_k), or (x_{k-1}, sigma_{k-1}) if
           psi rose in that last step (at the fp64 floor that comparison is
           roundoff, so it picks the iterate, never the count or the reason);
      (i)  otherwise, k >= 2 and psi_k > psi_{k-1} (>= under the weak rule,
           l.532): return (x_{k-1}, sigma_{k-1}); PSI_INCREASE_CONVERGED if the
           tol crossing already happened, else STAGNATED (status 7, R7);
      (iii) k > max_outer: MAX_OUTER (status 3)."""
    o = opts or RqiOptions()
    variant = "A" if o.op_variant == 0 else "paper"
    rule = "spec" if o.breakdown_rule == 0 else "paper"
    tol_in = tol if o.tol_inner <= 0 else o.tol_inner
    n = A.shape[1]
    A32 = A.astype(np.float32) if (o.u_p == "fp32" and variant == "A") else None   # fl32(A), RNE
    if pc.status != OK:
        return RqiResult(np.zeros(n), math.nan, pc.status, T_BREAKDOWN, 0, 0, [], [], [])
    if o.precond_apply == 2 and pc.W is None:
        pc = with_inverse(pc)
    passes = 0
    normAb2 = pc.normA2 + float(b @ b)
    h = rmatvec(A, b)                          # A^T b (setup pass)
    passes += 1
    # l.226  x_0 = x_LS  (R5: preconditioned CGLS = PCGTLS at sigma^2 = 0)
    if o.boot == 0:
        br = pcgtls(A, pc, 0.0, h, o.boot_max, o.boot_tol, "A", rule)
        x0, B0 = br.omega, br.count
        passes += 2 * br.count + (1 if br.count < o.boot_max else 0)
    else:
        x0, B0 = apply_Pinv(pc, apply_PinvT(pc, h)), 0
    r0 = b - matvec(A, x0)                     # l.227
    passes += 1
    sig0 = float(r0 @ r0) / (1.0 + float(x0 @ x0))   # l.229
    u0 = apply_Pinv(pc, apply_PinvT(pc, x0))   # l.233 (reading R9)
    x = x0 + sig0 * u0                         # l.235

    res = RqiResult(x, math.nan, OK, T_NONE, 0, B0, [], [], [])
    prev = None           # (x, sigma2) of step k-1
    psi_prev = None
    crossed_at = None
    k = 1
    while True:
        sig2, f, g, psi = newton_residual(A, b, x)
        passes += 1
        res.sigma2_trace.append(sig2)
        res.psi_trace.append(psi)
        res.rqi_iters = k
        if not (math.isfinite(sig2) and math.isfinite(psi)):
            res.x, res.sigma, res.status, res.termination = x, math.nan, NONFINITE, T_NONFINITE
            break
        increased = k >= 2 and (psi > psi_prev or (o.stop_rule == 1 and psi >= psi_prev))
        # (ii) tol crossing + polish (R6): the count is fixed by the crossing; at
        # the last polish step the better of x_k, x_{k-1} (by psi) is returned.
        if crossed_at is None and psi <= tol * normAb2:
            crossed_at = k
        if crossed_at is not None and k == crossed_at + o.polish:
            if increased:
                res.x, res.sigma = prev[0], math.sqrt(prev[1])
            else:
                res.x, res.sigma = x, math.sqrt(sig2)
            res.status, res.termination = OK, T_CONVERGED_TOL
            break
        # (i) psi increase (l.265)
        if increased:
            res.x, res.sigma = prev[0], math.sqrt(prev[1])
            if crossed_at is not None:
                res.status, res.termination = OK, T_PSI_INCREASE_CONVERGED
            else:
                res.status, res.termination = STAGNATED, T_STAGNATED
            break
        # (iii) cap
        if k > o.max_outer:
            res.x, res.sigma, res.status, res.termination = x, math.sqrt(sig2), MAX_OUTER, T_MAX_OUTER
            break
        budget = k + 1 if o.budget_rule == 0 else 400
        ra = pcgtls(A, pc, sig2, -f, budget, tol_in, variant, rule, A32)     # l.246
        rb = pcgtls(A, pc, sig2, x, budget, tol_in, variant, rule, A32)      # l.252
        if variant == "A":
            passes += ra.count + rb.count + (ra.breakdown or ra.count < budget) + (rb.breakdown or rb.count < budget)
        res.pcg_iters.append((ra.count, rb.count))
        res.delta_min_trace.append((ra.delta_min, rb.delta_min))
        if ra.breakdown or rb.breakdown:
            res.x, res.sigma = x, math.sqrt(sig2)
            res.status, res.termination = PCG_BREAKDOWN, T_BREAKDOWN
            res.breakdown_k = k
            res.breakdown_rhs = 0 if ra.breakdown else 1
            res.breakdown_j = ra.breakdown_j if ra.breakdown else rb.breakdown_j
            break
        z = x + ra.omega                       # l.248
        beta = (float(z @ f) - g) / (float(z @ x) + 1.0)   # l.250
        x_new = z + beta * rb.omega            # l.254
        prev, psi_prev = (x, sig2), psi
        x = x_new
        k += 1
    if res.status == OK and o.minimal_check > 0:                # R28
        nm, _ = minimality_certificate(A, pc, res.sigma ** 2, o.minimal_check)
        passes += o.minimal_check
        if nm:
            res.status = NOT_MINIMAL
    res.passes = passes
    return res


def _two_sum(a, b):
    """Knuth's TwoSum: s + e = a + b exactly (s = fl(a + b))."""
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def _split(a):
    """Veltkamp split of fp64 values into 26 + 27 significant bits."""
    c = 134217729.0 * a        # 2^27 + 1
    hi = c - (c - a)
    return hi, a - hi


def _two_prod(a, b):
    """Dekker's TwoProduct: p + e = a * b exactly (p = fl(a * b)), without an fma."""
    p = a * b
    ah, al = _split(a)
    bh, bl = _split(b)
    return p, al * bl - (((p - ah * bh) - al * bh) - ah * bl)


def dot2_rows(terms_a, terms_b):
    """Dot2 (Ogita, Rump & Oishi 2005, Alg. 5.3) of each row of two (rows x k) arrays,
    summed left to right: as accurate as the dot product in twice fp64 rounded once."""
    s = np.zeros(terms_a.shape[0])
    c = np.zeros(terms_a.shape[0])
    for j in range(terms_a.shape[1]):
        p, e = _two_prod(terms_a[:, j], terms_b[:, j])
        s, q = _two_sum(s, p)
        c = c + (q + e)
    return s + c


def certify_sigma(A, b: np.ndarray, x: np.ndarray) -> float:
    """The final certificate: sigma = sqrt(||b - A x||^2 /
    (1 + ||x||^2)) with r_i = b_i - a_i . x, ||r||^2 and ||x||^2 each formed by Dot2
    (compensated products and sums), then one fp64 square root of the quotient."""
    if _is_sparse(A):
        A = A.toarray()
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    # r_i = Dot2 over the n + 1 terms (b_i * 1) + sum_j (-a_ij) x_j
    ta = np.concatenate([b[:, None], -A], axis=1)
    tb = np.concatenate([np.ones((m, 1)), np.broadcast_to(x, (m, n))], axis=1)
    r = dot2_rows(ta, tb)
    rho = dot2_rows(r[None, :], r[None, :])[0]
    xx = dot2_rows(x[None, :], x[None, :])[0]
    return math.sqrt(rho / (1.0 + xx))


def solve(A, b, u_f: str, tol: float = 1e-14, opts: Optional[RqiOptions] = None):
    """Factor + RQI in one call (the whole hot path)."""
    o = opts or RqiOptions()
    pc = factor_precond(A, u_f, o.gram_chunk)
    return pc, rqi_pcgtls_mp(A, b, pc, tol, o)
