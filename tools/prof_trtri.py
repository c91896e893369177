"""Profiling driver: forming W = R~^{-1} (k_trtri) for n = 1024 and 2048 through tls_precond_apply.  Used under ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, tlsgen
from paper_2305_19028_b200 import tlsrqi as T
for n in (1024, 2048):
    P = tlsgen.dense_problem(8 * n, n, 1e3, 1e-3, 7, twin=True, device="cuda", keep_factors=False)
    M = T.matrix(P.A); ws = T.workspace(M)
    rc, R, _ = T.tls_factor_precond(M, "fp16", ws=ws)
    Y = torch.zeros((1, n), dtype=torch.float64, device="cuda")
    T.tls_precond_apply(R, 2, Y)
torch.cuda.synchronize()
