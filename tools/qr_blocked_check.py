"""GPU blocked QR (tls_factor_precond_qr_blocked, R29) against oracle.qr.householder_qr_r_blocked
and the unblocked R25 QR; timing against the unblocked GPU QR.

  python tools/qr_blocked_check.py [--time]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import rqi  # noqa: E402
from oracle.qr import householder_qr_r_blocked  # noqa: E402
from paper_2305_19028_b200 import tlsrqi as T  # noqa: E402


def ordered16(x, fmt):
    x = np.asarray(x, dtype=np.float64)
    if fmt == "fp16":
        b = x.astype(np.float16).view(np.int16).astype(np.int64)
        return np.where(b < 0, -(b & 0x7FFF), b)
    b = (x.astype(np.float32).view(np.int32).astype(np.int64)) >> 16
    return np.where(b < 0, -(b & 0x7FFF), b)


def problem(m, n, kappa, seed):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((m, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)))
    A = (U * np.logspace(0, -np.log10(kappa), n)) @ V.T
    return A * np.exp2(rng.integers(-4, 5, n))[None, :]


def main():
    for m, n, fmt in ((600, 128, "fp16"), (1100, 530, "fp16"), (2048, 256, "bf16"), (3000, 700, "fp16")):
        A = problem(m, n, 1e2, m + n)
        M = T.matrix(torch.as_tensor(A, device="cuda"))
        rc, R, info = T.tls_factor_precond_qr_blocked(M, fmt)
        print(f"{m}x{n} {fmt}: rc={rc}", flush=True)
        if R is None:
            continue
        Rt, d, nrm = T.tls_precond_export(R)
        d2, _ = rqi.norm_scaling(A)
        Rb = householder_qr_r_blocked(A / d2, fmt, 128)
        Ru = rqi.factor_precond_qr(A, fmt).Rt
        iu = np.triu_indices(n)
        same = np.mean(Rt[iu] == Rb[iu])
        ulps = np.abs(ordered16(Rt[iu], fmt) - ordered16(Rb[iu], fmt))
        print(f"   vs oracle R29: identical {same:.4f}, max ulps {ulps.max()}, >2 ulps {np.mean(ulps > 2):.4f}; "
              f"rel {np.linalg.norm(Rt - Rb) / np.linalg.norm(Rb):.2e}; vs unblocked rel {np.linalg.norm(Rt - Ru) / np.linalg.norm(Ru):.2e}; "
              f"d equal {np.array_equal(d, d2)}", flush=True)
    if "--time" in sys.argv:
        for m, n in ((16384, 1024), (65536, 2048)):
            A = torch.randn((m, n), dtype=torch.float64, device="cuda")
            M = T.matrix(A)
            for name, fn in (("blocked", T.tls_factor_precond_qr_blocked), ("unblocked", T.tls_factor_precond_qr)):
                fn(M, "fp16")
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(3):
                    rc, R, info = fn(M, "fp16")
                e1.record()
                torch.cuda.synchronize()
                print(f"{m}x{n} {name}: {e0.elapsed_time(e1) / 3:.2f} ms (rc {rc}, launches {info['launches']})", flush=True)


if __name__ == "__main__":
    main()
