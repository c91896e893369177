"""Where does the GPU's u_f Householder QR first differ from oracle.qr?  For each case prints
the first row j of R~ that differs, the differing columns and values, and the oracle's and
the GPU's diagonal there.  Run under several environments (TLS_QR_PDL=0).

  python tools/qr_diff.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import rqi  # noqa: E402
from paper_2305_19028_b200 import tlsrqi as T  # noqa: E402


def problem(m, n, kappa, seed):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((m, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = np.logspace(0, -np.log10(kappa), n)
    A = (U * s) @ V.T
    A = A * np.exp2(rng.integers(-6, 7, n))[None, :]
    return A


def main():
    cases = [(1100, 530, 1e2, "bf16", 1630), (1100, 530, 1e2, "fp16", 1630), (777, 67, 1e2, "bf16", 844),
             (600, 300, 1e2, "fp16", 900), (1100, 300, 1e2, "fp16", 1400), (1100, 400, 1e2, "fp16", 1500),
             (1100, 520, 1e2, "fp16", 1620)]
    for m, n, kappa, fmt, seed in cases:
        A = problem(m, n, kappa, seed)
        pc = rqi.factor_precond_qr(A, fmt)
        Ap = np.zeros((m, n + (n & 1)))
        Ap[:, :n] = A
        t = torch.as_tensor(Ap, device="cuda")
        M = T.matrix(t, n=n)
        rc, R, info = T.tls_factor_precond_qr(M, fmt)
        Rt, d, nrm = T.tls_precond_export(R)
        same_d = np.array_equal(d, pc.d)
        iu = np.triu_indices(n)
        frac = float(np.mean(Rt[iu] == pc.Rt[iu]))
        rows = [j for j in range(n) if not np.array_equal(Rt[j], pc.Rt[j])]
        msg = f"{m}x{n} {fmt} env PDL={os.environ.get('TLS_QR_PDL', '1')}: " \
              f"d equal {same_d}, identical {frac:.4f}"
        if rows:
            j = rows[0]
            cols = np.nonzero(Rt[j] != pc.Rt[j])[0]
            msg += f", first row {j}: {len(cols)} cols differ, first cols {cols[:6].tolist()}, " \
                   f"gpu {Rt[j, cols[:3]].tolist()} oracle {pc.Rt[j, cols[:3]].tolist()}, diag gpu {Rt[j, j]} or {pc.Rt[j, j]}"
        print(msg, flush=True)


if __name__ == "__main__":
    main()
