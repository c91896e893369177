"""Diagnose the tensor-core Gram at full cfg4w size: compare with the CUDA-core
fp32-chunk Gram and an fp64 Gram of the same rounded A^, and try fp64 Cholesky."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import tlsgen
from paper_2305_19028_b200 import tlsrqi

m = int(os.environ.get("GC_M", 1 << 20)); n = int(os.environ.get("GC_N", 1024))
P = tlsgen.dense_problem(m, n, 1e4, 1e-3, 4, twin=True, device="cuda", keep_factors=False)
M = tlsrqi.matrix(P.A)
ws = tlsrqi.workspace(M)
colmax, sumsq = tlsrqi.tls_colstats(M, ws=ws)
e = torch.frexp(colmax)[1]
d = torch.ldexp(torch.ones_like(colmax), e - 1)
Ah = (P.A / d).to(torch.float16).to(torch.float64)   # direct? torch double->half is RNE
G64 = (Ah.T @ Ah).cpu().numpy()
absG = (Ah.abs().T @ Ah.abs()).cpu().numpy()
for K_t in (2048, 256, 64):
    res = {}
    for path in ("tc", "cc"):
        if path == "cc": os.environ["TLS_GRAM"] = "cc"
        else: os.environ.pop("TLS_GRAM", None)
        torch.cuda.synchronize(); t = time.time()
        rc, G = tlsrqi.tls_gram(M, "fp16", d, K_t, ws=ws)
        torch.cuda.synchronize(); dt = time.time() - t
        G = G.cpu().numpy()
        err = np.abs(G - G64) / absG
        L = np.linalg.eigvalsh(G)
        res[path] = (dt, err.max(), np.median(err), L[0], L[-1])
        print(f"K_t={K_t} {path}: time {dt*1e3:.1f} ms  max rel err {err.max():.2e} median {np.median(err):.2e}  lam_min {L[0]:.3e} lam_max {L[-1]:.3e}", flush=True)
L = np.linalg.eigvalsh(G64)
print("fp64 Gram of A^: lam_min", L[0], "lam_max", L[-1])
