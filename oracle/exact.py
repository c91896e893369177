"""The definitional TLS result (oracle c1; test infrastructure).

PAPER.md §1 l.58-60: with the SVD [A, b] = U Sigma V^T, sigma_1 >= ... >= sigma_{n+1},
the TLS correction has norm sigma_{n+1} and
    x_TLS = -[v_{1,n+1}, ..., v_{n,n+1}]^T / v_{n+1,n+1}.
PAPER.md l.62: kappa_TLS = sigma'_1 / (sigma'_n - sigma_{n+1}), sigma' = singular
values of A.  PAPER.md l.268: x_TLS is unique if sigma'_n > sigma_{n+1}.
PAPER.md l.285-288 (constr1) and l.380-387 (constr2) give the u_q heuristics.
"""
from __future__ import annotations

import dataclasses

import math

import numpy as np


@dataclasses.dataclass
class TlsExact:
    sigma: float          # sigma_{n+1} of [A, b]
    x: np.ndarray         # x_TLS
    sigma_A_min: float    # sigma'_n
    sigma_A_max: float    # sigma'_1
    v_last: float         # v_{n+1,n+1}

    @property
    def kappa_tls(self) -> float:
        """PAPER.md l.62."""
        return self.sigma_A_max / (self.sigma_A_min - self.sigma)

    @property
    def unique(self) -> bool:
        """PAPER.md l.268."""
        return self.sigma_A_min > self.sigma and self.v_last != 0.0


def _from_right_vector(v: np.ndarray, sigma: float, sA: np.ndarray) -> TlsExact:
    n = v.shape[0] - 1
    x = -v[:n] / v[n]
    return TlsExact(float(sigma), x, float(sA[-1]), float(sA[0]), float(v[n]))


def tls_svd(A: np.ndarray, b: np.ndarray) -> TlsExact:
    """sigma_{n+1}, x_TLS from LAPACK SVD (gesdd) of the m x (n+1) matrix [A, b]."""
    C = np.column_stack([A, b])
    _, S, Vt = np.linalg.svd(C, full_matrices=False)
    sA = np.linalg.svd(A, compute_uv=False)
    return _from_right_vector(Vt[-1], S[-1], sA)


def tls_qr_svd(A: np.ndarray, b: np.ndarray) -> TlsExact:
    """Same result for tall [A, b]: Householder QR (geqrf) of [A, b], then the SVD
    of the (n+1) x (n+1) triangular factor (singular values and right singular
    vectors are invariant under the orthogonal Q)."""
    C = np.column_stack([A, b])
    Rf = np.linalg.qr(C, mode="r")
    _, S, Vt = np.linalg.svd(Rf)
    sA = np.linalg.svd(Rf[:-1, :-1], compute_uv=False)
    return _from_right_vector(Vt[-1], S[-1], sA)


def tls_arrow(s: np.ndarray, V: np.ndarray, c: np.ndarray, rho: float) -> TlsExact:
    """Reduced model for A = U diag(s) V^T (U orthonormal columns):
    with c = U^T b and rho = ||b - U c||, [A, b] = [U, q] K diag(V, 1)^T with
    K = [[diag(s), c], [0, rho]], so [A, b] has the singular values of K and right
    singular vectors diag(V, 1) w.  Independent of the m-dimensional SVD."""
    n = s.shape[0]
    K = np.zeros((n + 1, n + 1))
    K[np.arange(n), np.arange(n)] = s
    K[:n, n] = c
    K[n, n] = rho
    _, S, Wt = np.linalg.svd(K)
    w = Wt[-1]
    v = np.concatenate([V @ w[:n], [w[n]]])
    sA = np.sort(s)[::-1]
    return _from_right_vector(v, S[-1], sA)


def constraints(A: np.ndarray, ex: TlsExact) -> dict:
    """u_q heuristics: constr1 u_q <~ 1/kappa(A) (l.285-288) and
    constr2 u_q <~ kappa_F(A)^-1 (1 - sigma_{n+1}^2/sigma'_n^2) (l.380-387),
    with kappa_F(A) = ||A||_F / sigma'_n (reading R13)."""
    kappa = ex.sigma_A_max / ex.sigma_A_min
    kappa_F = np.linalg.norm(A) / ex.sigma_A_min
    gap = 1.0 - ex.sigma ** 2 / ex.sigma_A_min ** 2
    return {"kappa": kappa, "kappa_F": kappa_F, "gap": gap,
            "constr1": 1.0 / kappa, "constr2": gap / kappa_F}


def constraint_report(m: int, n: int, sigma_A: np.ndarray, sigma: float, normF: float,
                      lam_min_H: float, c: float = 1.0) -> dict:
    """All the factorization-precision constraints of PAPER.md §3.1 (l.270-391), c = 1
    (reading R13), from the singular values of A, sigma_{n+1}, ||A||_F and lambda_min(H):
      D1  u_q < 1/(c m n^{3/2} kappa)              QR: R^ nonsingular (l.279-281)
      D2  u_q < 1/(c m^{1/2} n^{3/4} kappa)        the probabilistic version (l.283-286)
      D3  u_q <~ 1/kappa                           constr1 (l.287-288)
      D4  u_q <= 1/(20 n^{3/2} kappa^2)            Cholesky of fl(A^T A), Wilkinson (l.290-294)
      D5  u_q <~ 1/kappa^2                         its heuristic (l.295-296)
      D6  u_q < lmin(H)/((2 lmin(H) + n)(n + 1))   scaled Cholesky, H = D^{-1} fl(A^TA) D^{-1} (l.298-304)
      D7  sqrt(m) g_mn kappa_F < gap, g_mn = c m n u/(1 - c m n u): positive-definite C^ (l.364-378)
      D8  u_q <~ gap / kappa_F                     constr2 (l.386-387)
    with gap = 1 - sigma_{n+1}^2/sigma'_n^2 and kappa_F = ||A||_F / sigma'_n."""
    smax, smin = float(np.max(sigma_A)), float(np.min(sigma_A))
    kappa = smax / smin
    kappa_F = normF / smin
    gap = 1.0 - sigma * sigma / (smin * smin)
    g = gap / (math.sqrt(m) * kappa_F)           # D7: c m n u / (1 - c m n u) < g
    return {"kappa": kappa, "kappa_F": kappa_F, "gap": gap,
            "D1": 1.0 / (c * m * n ** 1.5 * kappa),
            "D2": 1.0 / (c * math.sqrt(m) * n ** 0.75 * kappa),
            "D3": 1.0 / kappa,
            "D4": 1.0 / (20.0 * n ** 1.5 * kappa * kappa),
            "D5": 1.0 / (kappa * kappa),
            "D6": lam_min_H / ((2.0 * lam_min_H + n) * (n + 1)),
            "D7": (g / (c * m * n * (1.0 + g))) if g > 0 else 0.0,
            "D8": gap / kappa_F}


def lam_min_H(A: np.ndarray) -> float:
    """lambda_min of H = D^{-1} A^T A D^{-1}, D = diag(A^T A)^{1/2}."""
    G = A.T @ A
    dd = 1.0 / np.sqrt(np.diag(G))
    return float(np.linalg.eigvalsh(G * dd[:, None] * dd[None, :])[0])


def rayleigh_sigma2(A: np.ndarray, b: np.ndarray, x: np.ndarray) -> float:
    """||[A, b][x; -1]||^2 / (1 + ||x||^2): equals
    sigma_{n+1}^2 at x = x_TLS."""
    r = b - A @ x
    return float(r @ r / (1.0 + x @ x))
