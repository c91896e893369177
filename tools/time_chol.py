"""Device time of the preconditioner build pieces for n in {1024, 2000, 2048} (m = 4n):
the whole tls_factor_precond per call (CUDA events), and R~ vs the oracle's LAPACK factor."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2305_19028_b200 import tlsrqi
from oracle import rqi
for n in (1024, 2000, 2048):
    m = 8 * n
    rng = np.random.default_rng(0)
    A_np = rng.standard_normal((m, n)) * np.logspace(0, -2, n)[None, :]
    A = torch.as_tensor(A_np, device="cuda")
    M = tlsrqi.matrix(A)
    ws = tlsrqi.workspace(M)
    tlsrqi.tls_profile_enable(True)
    rc, R, fi = tlsrqi.tls_factor_precond(M, "fp16", ws=ws)
    for _ in range(3):
        rc, R, fi = tlsrqi.tls_factor_precond(M, "fp16", ws=ws)
    prof = tlsrqi.tls_profile_read()
    tlsrqi.tls_profile_enable(False)
    Rt, d, _ = tlsrqi.tls_precond_export(R)
    pc = rqi.factor_precond(A_np, "fp16")
    ulp = np.spacing(np.abs(pc.Rt).astype(np.float16)).astype(np.float64)
    frac = np.mean(np.abs(Rt - pc.Rt) <= ulp)
    print(f"n={n}: chol {prof['chol']['ms'] / prof['chol']['count']:.3f} ms  gram {prof['gram']['ms'] / prof['gram']['count']:.3f} ms"
          f"  R~ within 1 ulp of oracle: {frac * 100:.3f}%  max |diff|/ulp {np.max(np.abs(Rt - pc.Rt) / ulp):.2f}", flush=True)
