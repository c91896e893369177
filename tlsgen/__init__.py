"""Seeded synthetic TLS problem generators (shared by the oracle tests, the GPU
parity tests and bench.py).

This module holds NO arithmetic of the RQI-PCGTLS-MP method: it only draws
random numbers and builds the input matrices A, b of BASELINE.json's configs
(DESIGN.md "Input recipe").  The oracle (oracle/) and the CUDA path
(paper_2305_19028_b200/) both consume the bytes produced here and nothing else
from each other.

Construction (BASELINE.json configs[0..4]):
  A = U diag(s) V^T,  U (m x n) orthonormalised Gaussian (Householder QR of a
  Gaussian, columns sign-fixed so diag(R) > 0), V (n x n) the same ("Haar"),
  s = logspace(0, -log10(kappa), n), x_true ~ N(0, I), g ~ N(0, I),
  b = A x_true + eps * g            (literal configs)
  b = A x_true + eps * g / sqrt(m)  ("w" twins, reading R8)
A is returned row-major (C-contiguous) fp64, which is the layout the C ABI
takes (include/tlsrqi.h, TLS_DENSE_ROWMAJOR).

Draw order (fixed): G_U (m*n), G_V (n*n), x_true (n), g (m).
CPU generation uses numpy Generator(PCG64(seed)); the large configs (cfg4,
cfg5 at full size) are generated on a CUDA device with torch's seeded Philox
generator + torch.linalg.qr, because a host QR of a 2^20 x 1024 matrix takes
minutes.  Either way the oracle and the GPU read the same bytes.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

__all__ = [
    "DenseProblem", "CsrProblem", "dense_problem", "csr_problem", "ragged_csr", "config",
    "CONFIGS",
]


@dataclasses.dataclass
class DenseProblem:
    name: str
    A: object            # (m, n) float64 row-major; numpy array or torch tensor
    b: object            # (m,) float64
    x_true: object       # (n,)
    s: np.ndarray        # (n,) singular values of A by construction
    V: Optional[object]  # (n, n) right singular vectors of A (small cases)
    U: Optional[object]  # (m, n) left singular vectors (small cases only)
    kappa: float
    eps: float
    twin: bool
    seed: int
    u_f: str = "fp16"
    c: Optional[np.ndarray] = None   # U^T b (reduced "arrow" model, oracle/exact.py)
    rho: Optional[float] = None      # ||b - U U^T b||

    @property
    def m(self) -> int:
        return int(self.A.shape[0])

    @property
    def n(self) -> int:
        return int(self.A.shape[1])


@dataclasses.dataclass
class CsrProblem:
    name: str
    m: int
    n: int
    rowptr: np.ndarray   # (m+1,) int64
    colidx: np.ndarray   # (nnz,) int32, sorted within each row
    vals: np.ndarray     # (nnz,) float64
    b: np.ndarray        # (m,)
    x_true: np.ndarray   # (n,)
    eps: float
    seed: int
    u_f: str = "fp16"

    def to_dense(self) -> np.ndarray:
        A = np.zeros((self.m, self.n))
        rows = np.repeat(np.arange(self.m), np.diff(self.rowptr))
        A[rows, self.colidx] = self.vals
        return A


def _orthonormal_np(G: np.ndarray) -> np.ndarray:
    Q, R = np.linalg.qr(G, mode="reduced")
    sgn = np.sign(np.diag(R))
    sgn[sgn == 0] = 1.0
    return Q * sgn[None, :]


def dense_problem(m: int, n: int, kappa: float, eps: float, seed: int,
                  twin: bool = False, device: str = "cpu", name: str = "",
                  u_f: str = "fp16", keep_factors: Optional[bool] = None) -> DenseProblem:
    """Build A = U diag(s) V^T and b = A x_true + noise (module docstring).

    device="cpu": numpy arrays; device="cuda[:i]": torch tensors on that device.
    keep_factors: return U and V (default: only when m*n <= 2^22).
    """
    if keep_factors is None:
        keep_factors = m * n <= (1 << 22)
    s = np.logspace(0.0, -math.log10(kappa), n)
    scale = eps / math.sqrt(m) if twin else eps
    if device == "cpu":
        rng = np.random.Generator(np.random.PCG64(seed))
        GU = rng.standard_normal((m, n))
        GV = rng.standard_normal((n, n))
        x_true = rng.standard_normal(n)
        g = rng.standard_normal(m)
        U = _orthonormal_np(GU)
        del GU
        V = _orthonormal_np(GV)
        A = np.ascontiguousarray((U * s[None, :]) @ V.T)
        b = A @ x_true + scale * g
        c = U.T @ b
        rho = float(np.linalg.norm(b - U @ c))
        return DenseProblem(name, A, b, x_true, s, V if keep_factors else None,
                            U if keep_factors else None, kappa, eps, twin, seed, u_f, c, rho)
    import torch
    dev = torch.device(device)
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    GU = torch.randn((m, n), generator=gen, dtype=torch.float64, device=dev)
    GV = torch.randn((n, n), generator=gen, dtype=torch.float64, device=dev)
    x_true = torch.randn((n,), generator=gen, dtype=torch.float64, device=dev)
    g = torch.randn((m,), generator=gen, dtype=torch.float64, device=dev)
    U, R = torch.linalg.qr(GU, mode="reduced")
    del GU
    sg = torch.sign(torch.diagonal(R))
    sg[sg == 0] = 1.0
    U.mul_(sg[None, :])
    del R
    V, RV = torch.linalg.qr(GV, mode="reduced")
    sv = torch.sign(torch.diagonal(RV))
    sv[sv == 0] = 1.0
    V = V * sv[None, :]
    st = torch.as_tensor(s, dtype=torch.float64, device=dev)
    A = U @ (st[:, None] * V.T)
    A = A.contiguous()
    b = A @ x_true + scale * g
    c = U.T @ b
    rho = float(torch.linalg.norm(b - U @ c))
    c = c.cpu().numpy()
    if not keep_factors:
        del U
        U = None
    return DenseProblem(name, A, b, x_true, s, V.cpu().numpy(), U, kappa, eps, twin, seed, u_f,
                        c, rho)


def csr_problem(m: int = 200000, n: int = 2000, per_row: int = 10, eps: float = 1e-3,
                seed: int = 3, name: str = "cfg3", u_f: str = "fp16") -> CsrProblem:
    """BASELINE.json configs[2]: each row i holds `per_row` DISTINCT columns drawn
    uniformly from {0..n-1} minus {i mod n}, plus column i mod n (DESIGN.md
    reading R16); values N(0,1); columns sorted; b = A x_true + eps*g.
    Draw order: per row the column sample, then all values, then x_true, g."""
    rng = np.random.Generator(np.random.PCG64(seed))
    cols = np.empty((m, per_row + 1), dtype=np.int64)
    diag = np.arange(m) % n
    # Distinct draws by whole-row rejection: draw per_row values in [0, n-1);
    # redraw every row that holds a duplicate; then shift values >= i mod n by
    # one so the fixed column is never drawn.
    cand = rng.integers(0, n - 1, size=(m, per_row))
    while True:
        srt = np.sort(cand, axis=1)
        dup = (srt[:, 1:] == srt[:, :-1]).any(axis=1)
        if not dup.any():
            break
        cand[dup] = rng.integers(0, n - 1, size=(int(dup.sum()), per_row))
    cand = cand + (cand >= diag[:, None])
    cols[:, :per_row] = cand
    cols[:, per_row] = diag
    cols.sort(axis=1)
    vals = rng.standard_normal(m * (per_row + 1))
    x_true = rng.standard_normal(n)
    g = rng.standard_normal(m)
    rowptr = np.arange(0, m * (per_row + 1) + 1, per_row + 1, dtype=np.int64)
    colidx = cols.reshape(-1).astype(np.int32)
    # b = A x_true + eps g, A applied row by row from the CSR arrays
    prod = (vals * x_true[colidx]).reshape(m, per_row + 1).sum(axis=1)
    b = prod + eps * g
    return CsrProblem(name, m, n, rowptr, colidx, vals, b, x_true, eps, seed, u_f)


def ragged_csr(m: int, n: int, max_per_row: int, seed: int, eps: float = 1e-3,
               empty_frac: float = 0.05, name: str = "ragged") -> CsrProblem:
    """Edge-case CSR stand-in (tests only): row lengths uniform in [0, max_per_row]
    (a fraction `empty_frac` of rows empty), distinct sorted columns, values N(0,1)
    scaled by 10^U(-2,2) per row, plus one entry in every column (row j mod m) so
    no column is empty.  Draw order: lengths, per-row columns, values, scales,
    x_true, g."""
    rng = np.random.Generator(np.random.PCG64(seed))
    lens = rng.integers(0, max_per_row + 1, size=m)
    lens[rng.random(m) < empty_frac] = 0
    rows = []
    for i in range(m):
        rows.append(set(rng.choice(n, int(lens[i]), replace=False).tolist()) if lens[i] else set())
    for j in range(n):
        rows[j % m].add(j)
    lens = np.array([len(r) for r in rows], dtype=np.int64)
    rowptr = np.zeros(m + 1, dtype=np.int64)
    rowptr[1:] = np.cumsum(lens)
    colidx = np.concatenate([np.array(sorted(r), dtype=np.int32) for r in rows if r]).astype(np.int32)
    vals = rng.standard_normal(int(rowptr[-1]))
    scale = 10.0 ** rng.uniform(-2, 2, size=m)
    vals = vals * np.repeat(scale, lens)
    x_true = rng.standard_normal(n)
    g = rng.standard_normal(m)
    prod = np.zeros(m)
    np.add.at(prod, np.repeat(np.arange(m), lens), vals * x_true[colidx])
    b = prod + eps * g
    return CsrProblem(name, m, n, rowptr, colidx, vals, b, x_true, eps, seed)


# name -> (m, n, kappa, eps, seed, twin, u_f); cfg3 (CSR) handled separately.
CONFIGS = {
    "cfg1": (200, 20, 1e2, 1e-4, 1, False, "fp16"),
    "cfg2": (4096, 512, 1e3, 1e-3, 2, False, "bf16"),
    "cfg2w": (4096, 512, 1e3, 1e-3, 2, True, "bf16"),
    "cfg4": (1 << 20, 1024, 1e4, 1e-3, 4, False, "fp16"),
    "cfg4w": (1 << 20, 1024, 1e4, 1e-3, 4, True, "fp16"),
}


def config(name: str, device: str = "cpu", **kw):
    """Build one of BASELINE.json's configs by name.

    cfg5 cells are named "cfg5:k1e4:e1e-6" (kappa, eps); u_f is chosen by the caller.
    Scaled-down stand-ins keep the recipe: pass m=..., n=... to override sizes.
    """
    if name == "cfg3":
        return csr_problem(**kw)
    if name.startswith("cfg5"):
        fields = name.split(":")
        kappa = float(fields[1][1:]) if len(fields) > 1 else 1e4
        eps = float(fields[2][1:]) if len(fields) > 2 else 1e-6
        m = kw.pop("m", 65536)
        n = kw.pop("n", 2048)
        return dense_problem(m, n, kappa, eps, 5, twin=False, device=device, name=name,
                             u_f=kw.pop("u_f", "fp16"), **kw)
    m, n, kappa, eps, seed, twin, u_f = CONFIGS[name]
    m = kw.pop("m", m)
    n = kw.pop("n", n)
    return dense_problem(m, n, kappa, eps, seed, twin=twin, device=device, name=name,
                         u_f=kw.pop("u_f", u_f), **kw)


# --------------------------------------------------------------------------- PAPER §4 problems
@dataclasses.dataclass
class PaperProblem:
    """One of the paper's §4 test problems, as (A+E, b+e)."""
    name: str
    A: np.ndarray        # (m, n) float64 row-major: the perturbed A + E
    b: np.ndarray        # (m,) the perturbed b + e
    A0: np.ndarray       # unperturbed A
    b0: np.ndarray       # unperturbed b
    x_true: Optional[np.ndarray]
    eps: float
    seed: int
    u_f: str = "fp16"

    @property
    def m(self) -> int:
        return int(self.A.shape[0])

    @property
    def n(self) -> int:
        return int(self.A.shape[1])


def _haar(k: int, rng) -> np.ndarray:
    return _orthonormal_np(rng.standard_normal((k, k)))


def paper_problem(name: str, seed: int = 1, eps: Optional[float] = None, **kw) -> PaperProblem:
    """The five §4 problems with the paper's sizes and noise levels.  numpy's PCG64 stands
    in for MATLAB's rng (SURVEY.md §8(f) OUT OF SCOPE: RNG-exact reproduction), so the
    instances are the paper's distributions, not its bytes (R20-R22).

      random     PAPER.md:484-487  A = rand(100,60), b = ones, E = eps rand, e = eps rand, eps 1e-6
      delta      PAPER.md:501-531  the 9x4 pattern (delta at (1,1),(3,2); 1 at (7,3),(9,4)),
                                   b = ones, E = eps Ebar .* A, e = eps ebar .* b with Ebar,
                                   ebar ~ U(-1,1); eps 1e-1, delta 1e-2
      bjorck     PAPER.md:539-550  A = Y [D; 0] Z^T, D = diag(2^0..2^-(n-1)), (m,n) = (30,15),
                                   x = (1, 1/2, .., 1/n), b = A x; E = eps rand, e = eps rand, eps 0.05
      toeplitz   PAPER.md:572-587  Tbar (n x n-2w) lower banded Toeplitz with first column
                                   t_i = exp(-(w-i+1)^2/(2 a^2))/sqrt(2 pi a^2), i = 1..2w+1;
                                   E = toeplitz(c, r) random (c ~ U(0,1)^n, r = (c_1, U(0,1)..));
                                   b = ones + e; E, e scaled by 1e-3; n 100, w 2, a 1.25
      vanhuffel  PAPER.md:591-604  n x (n-2): n-1 on the diagonal of the top (n-2) block, -1
                                   elsewhere; b = (-1,..,-1, n-1, -1); E = eps rand, e = eps rand,
                                   eps 1e-6, n 100
    Draw order per problem: the matrices named above, then E, then e.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    x_true = None
    if name == "random":
        m, n = kw.get("m", 100), kw.get("n", 60)
        eps = 1e-6 if eps is None else eps
        A0 = rng.random((m, n))
        b0 = np.ones(m)
        E = eps * rng.random((m, n))
        e = eps * rng.random(m)
    elif name == "delta":
        delta = kw.get("delta", 1e-2)
        eps = 1e-1 if eps is None else eps
        A0 = np.zeros((9, 4))
        A0[0, 0] = delta
        A0[2, 1] = delta
        A0[6, 2] = 1.0
        A0[8, 3] = 1.0
        b0 = np.ones(9)
        E = eps * rng.uniform(-1.0, 1.0, (9, 4)) * A0
        e = eps * rng.uniform(-1.0, 1.0, 9) * b0
    elif name == "bjorck":
        m, n = kw.get("m", 30), kw.get("n", 15)
        eps = 0.05 if eps is None else eps
        Y = _haar(m, rng)
        Z = _haar(n, rng)
        D = np.zeros((m, n))
        D[np.arange(n), np.arange(n)] = 2.0 ** -np.arange(n)
        A0 = Y @ D @ Z.T
        x_true = 1.0 / np.arange(1, n + 1)
        b0 = A0 @ x_true
        E = eps * rng.random((m, n))
        e = eps * rng.random(m)
    elif name == "toeplitz":
        n, w, a = kw.get("n", 100), kw.get("omega", 2), kw.get("alpha", 1.25)
        eps = 1e-3 if eps is None else eps
        nc = n - 2 * w
        i = np.arange(1, 2 * w + 2)
        col = np.zeros(n)
        col[:2 * w + 1] = np.exp(-((w - i + 1) ** 2) / (2 * a * a)) / math.sqrt(2 * math.pi * a * a)
        idx = np.arange(n)[:, None] - np.arange(nc)[None, :]
        A0 = np.where(idx >= 0, col[np.clip(idx, 0, n - 1)], 0.0)
        c = rng.random(n)
        r = np.concatenate([[c[0]], rng.random(nc - 1)])
        E = eps * np.where(idx >= 0, c[np.clip(idx, 0, n - 1)], r[np.clip(-idx, 0, nc - 1)])
        b0 = np.ones(n)
        e = eps * rng.random(n)
    elif name == "vanhuffel":
        n = kw.get("n", 100)
        eps = 1e-6 if eps is None else eps
        A0 = -np.ones((n, n - 2))
        A0[np.arange(n - 2), np.arange(n - 2)] = n - 1.0
        b0 = -np.ones(n)
        b0[n - 2] = n - 1.0
        E = eps * rng.random((n, n - 2))
        e = eps * rng.random(n)
    else:
        raise ValueError(f"unknown paper problem {name!r}")
    A = np.ascontiguousarray(A0 + E)
    return PaperProblem(name, A, b0 + e, A0, b0, x_true, float(eps), seed)


PAPER_PROBLEMS = ("random", "delta", "bjorck", "toeplitz", "vanhuffel")
