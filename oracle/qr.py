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
