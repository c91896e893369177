"""Householder QR computed in a low precision u_q (oracle; TEST INFRASTRUCTURE ONLY, see
oracle/__init__.py).  Groundwork for SURVEY §8(f) NEXT-2: the paper's preferred
preconditioner is the R factor of a Householder QR of A computed in precision u_q
("Compute A = Q[R 0]^T in u_q", l.276-288); the GPU path of
this round uses the Cholesky of the u_f Gram instead (DESIGN R10).

The arithmetic follows the textbook algorithm (Golub & Van Loan Alg. 5.1.1 / Higham
§19.1) with every elementary vector operation rounded to u_q, the way the paper's
`chop` simulation rounds every operation (SPEC.md householder_qr):
for j = 0 .. n-1 (x = A[j:, j]):
    sigma = fl(||x||)             (dot product rounded, then a rounded square root)
    alpha = -sign(x_0) sigma       (the sign that avoids cancellation)
    v = x - alpha e_0, rounded;   beta = fl(2 / fl(v^T v))
    A[j:, j:] -= v (beta (v^T A[j:, j:]))   each of the three steps rounded
and R is the upper triangle with its rows' signs flipped so that diag(R) >= 0 (SPEC.md
"Sign convention").  Q is never formed.  Reading (R25): inner products are accumulated
in fp64 and rounded once (a wide accumulator, as on tensor cores), every elementwise
operation is rounded on its own.
"""
from __future__ import annotations

import numpy as np

from .rounding import round_to


class ZeroColumn(ZeroDivisionError):
    """Column `col` (0-based) is exactly zero below its diagonal position in fmt."""

    def __init__(self, col: int):
        super().__init__(f"zero column {col}")
        self.col = col


def householder_qr_r(A: np.ndarray, fmt: str, leaf: bool = False) -> np.ndarray:
    """R (n x n, upper, diag >= 0) of the Householder QR of A with every operation
    rounded to fmt.  A is first rounded to fmt.  Raises ZeroDivisionError on an exactly
    zero column (rank deficiency, SPEC.md householder_qr errors).
    leaf=True (a TSQR leaf, reading R26): a column that vanishes on this block's rows is
    not a rank deficiency of A (other blocks hold its mass), so its reflector is the
    identity H = I (nothing is applied) and R's row j is W[j, j:] as it stands (R_jj = 0);
    only the stack factorization reports a vanishing column."""
    rd = lambda x: round_to(np.asarray(x, dtype=np.float64), fmt)
    W = rd(np.array(A, dtype=np.float64, copy=True))
    m, n = W.shape
    if m < n:
        raise ValueError("householder_qr_r needs m >= n")
    for j in range(n):
        x = W[j:, j]
        sigma = float(rd(np.sqrt(rd(np.dot(x, x)))))
        if sigma == 0.0:
            if not leaf:
                raise ZeroColumn(j)
            continue                                   # H = I; row j of R is W[j, j:]
        alpha = -sigma if x[0] >= 0 else sigma
        v = x.copy()
        v[0] = float(rd(x[0] - alpha))
        vv = float(rd(np.dot(v, v)))
        beta = float(rd(2.0 / vv))
        # W[j:, j:] -= v (beta (v^T W[j:, j:]))
        wT = rd(v @ W[j:, j:])
        wT = rd(beta * wT)
        W[j:, j:] = rd(W[j:, j:] - rd(np.outer(v, wT)))
        W[j, j] = alpha
        W[j + 1:, j] = 0.0
    R = np.triu(W[:n, :n])
    sgn = np.where(np.diag(R) < 0, -1.0, 1.0)
    return R * sgn[:, None]


def tsqr_r(A: np.ndarray, row_blocks, fmt: str) -> np.ndarray:
    """TSQR (tall-skinny QR, reading R26): the R factors R_b of the row blocks A[r0:r1] (each a
    Householder QR in fmt, householder_qr_r) stacked row-interleaved -- stack row i B + b is
    row i of R_b -- then the R factor of that stack, again by householder_qr_r.  In exact
    arithmetic this is the R of A (diag >= 0): A = diag(Q_b) Pi S and S = Q' R for the row
    permutation Pi.  The interleaving puts every row whose first nonzero is in column i
    before those starting later, so the stack's column j only involves its first (j+1) B rows
    (the rest are zero and stay zero).  One block is the plain QR."""
    if len(row_blocks) == 1:
        r0, r1 = row_blocks[0]
        return householder_qr_r(A[r0:r1], fmt)
    Rs = [householder_qr_r(A[r0:r1], fmt, leaf=True) for r0, r1 in row_blocks]
    B, n = len(Rs), A.shape[1]
    S = np.zeros((B * n, n))
    for b, R in enumerate(Rs):
        S[b::B] = R
    return householder_qr_r(S, fmt)


def even_row_blocks(m: int, k: int):
    """k contiguous row ranges [s m // k, (s + 1) m // k): the split of a row block into k
    TSQR leaves (tlsrqi.h tls_factor_precond_qr)."""
    return [(s * m // k, (s + 1) * m // k) for s in range(k)]


# ----------------------------------------------------------------------------- blocked (R29)
def _fp32_seq_chunks(X: np.ndarray, Y: np.ndarray, chunk: int = 64) -> np.ndarray:
    """X^T Y (X: r x a, Y: r x c, u_f values) as reading R29 (= R11's Gram accumulation) sums it:
    the exact products of every `chunk` consecutive rows accumulated in fp32, one row at a time in
    row order, round to nearest; the chunk sums added in fp64 in chunk order."""
    r = X.shape[0]
    out = np.zeros((X.shape[1], Y.shape[1]))
    X32, Y32 = X.astype(np.float32), Y.astype(np.float32)
    for c0 in range(0, r, chunk):
        acc = np.zeros((X.shape[1], Y.shape[1]), dtype=np.float32)
        for i in range(c0, min(r, c0 + chunk)):
            acc = acc + np.outer(X32[i], Y32[i])         # exact products (u_f x u_f fits fp32), RNE add
        out += acc.astype(np.float64)
    return out


def _fp32_seq_matmul(V: np.ndarray, Y: np.ndarray) -> np.ndarray:
    """V Y (V: r x b, Y: b x c, u_f values) accumulated in fp32 over the b terms in order (RNE)."""
    V32, Y32 = V.astype(np.float32), Y.astype(np.float32)
    acc = np.zeros((V.shape[0], Y.shape[1]), dtype=np.float32)
    for j in range(V.shape[1]):
        acc = acc + np.outer(V32[:, j], Y32[j])
    return acc.astype(np.float64)


def householder_qr_r_blocked(A: np.ndarray, fmt: str, b: int = 128) -> np.ndarray:
    """R of the Householder QR of A in u_f with the trailing updates blocked (reading R29, SURVEY
    §8(f) NEXT-2 "on tensor cores"): panels of b columns, each factored by R25's unblocked
    Householder steps restricted to the panel, then the panel's b reflectors applied to the
    trailing columns C at once in compact WY form, C <- C - V (T^T (V^T C)), with
      V^T C, V^T V   exact u_f products, fp32 sums per 64-row chunk (in row order, RNE), the
                     chunk sums in fp64 (R11's accumulation: what the tensor cores compute),
      T              the upper-triangular WY factor in fp64: T_jj = beta_j,
                     T[0:j, j] = -beta_j T[0:j, 0:j] (V^T V)[0:j, j],
      Y = fl_uf(T^T (V^T C))        (fp64 product, rounded once to u_f),
      C <- fl_uf(C - fl32(V Y))     (V Y: exact products summed in fp32 over the b terms in
                                     order; the difference in fp64, rounded once to u_f).
    In exact arithmetic this is the unblocked factorization (compact WY, Schreiber & Van Loan);
    with b >= n it IS householder_qr_r.  u_f in {fp16, bf16} (the tensor-core formats); for
    fp32 / fp64 every fp32 sum above is replaced by fp64 (the fp64 control)."""
    rd = lambda x: round_to(np.asarray(x, dtype=np.float64), fmt)
    low = fmt in ("fp16", "bf16")
    W = rd(np.array(A, dtype=np.float64, copy=True))
    m, n = W.shape
    if m < n:
        raise ValueError("householder_qr_r_blocked needs m >= n")
    for c0 in range(0, n, b):
        c1 = min(n, c0 + b)
        nb = c1 - c0
        V = np.zeros((m - c0, nb))
        beta = np.zeros(nb)
        for j in range(c0, c1):                       # R25 on the panel columns only
            x = W[j:, j]
            sigma = float(rd(np.sqrt(rd(np.dot(x, x)))))
            if sigma == 0.0:
                raise ZeroColumn(j)
            alpha = -sigma if x[0] >= 0 else sigma
            v = x.copy()
            v[0] = float(rd(x[0] - alpha))
            vv = float(rd(np.dot(v, v)))
            bt = float(rd(2.0 / vv))
            if j + 1 < c1:
                wT = rd(bt * rd(v @ W[j:, j + 1:c1]))
                W[j:, j + 1:c1] = rd(W[j:, j + 1:c1] - rd(np.outer(v, wT)))
            W[j, j] = alpha
            W[j + 1:, j] = 0.0
            V[j - c0:, j - c0] = v
            beta[j - c0] = bt
        if c1 == n:
            break
        C = W[c0:, c1:]
        VtC = _fp32_seq_chunks(V, C) if low else V.T @ C
        VtV = _fp32_seq_chunks(V, V) if low else V.T @ V
        T = np.zeros((nb, nb))
        for j in range(nb):
            T[j, j] = beta[j]
            if j:
                T[:j, j] = -beta[j] * (T[:j, :j] @ VtV[:j, j])
        Y = rd(T.T @ VtC)
        VY = _fp32_seq_matmul(V, Y) if low else V @ Y
        W[c0:, c1:] = rd(C - VY)
    R = np.triu(W[:n, :n])
    sgn = np.where(np.diag(R) < 0, -1.0, 1.0)
    return R * sgn[:, None]
