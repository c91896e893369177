"""The paper's performance model (§3.2, l.404-417; test infrastructure
and reporting only — "model only, no hardware").

cost(m,n,r,c,c_p,c_q) = c  (2mn + 3m + 4n + 2n^2 - 2 + r(4mn + 5m + 11n - 5))
                      + c_p(2r(n^2 + 2n - 1) + (r^2 + 3r)(2n^2 + 14n - 3))
                      + c_q(2mn^2 - 2n^3/3)                          (l.410-412)
constants 1 / 0.5 / 0.25 for double / single / half (l.407).
The printed ratio (l.414-417) is MP/uniform; the speedup is read as
uniform/MP (reading R14).
"""
from fractions import Fraction

WEIGHT = {"fp64": Fraction(1), "fp32": Fraction(1, 2), "fp16": Fraction(1, 4),
          "bf16": Fraction(1, 4)}


def cost(m: int, n: int, r: int, c, c_p, c_q) -> Fraction:
    c, c_p, c_q = Fraction(c), Fraction(c_p), Fraction(c_q)
    t1 = 2 * m * n + 3 * m + 4 * n + 2 * n * n - 2 + r * (4 * m * n + 5 * m + 11 * n - 5)
    t2 = 2 * r * (n * n + 2 * n - 1) + (r * r + 3 * r) * (2 * n * n + 14 * n - 3)
    t3 = Fraction(2 * m * n * n) - Fraction(2 * n ** 3, 3)
    return c * t1 + c_p * t2 + c_q * t3


def speedup(m: int, n: int, r: int, u: str = "fp64", u_p: str = "fp32", u_q: str = "fp16") -> float:
    """uniform (1,1,1) cost over mixed-precision cost (R14)."""
    mp = cost(m, n, r, WEIGHT[u], WEIGHT[u_p], WEIGHT[u_q])
    uni = cost(m, n, r, 1, 1, 1)
    return float(uni / mp)
