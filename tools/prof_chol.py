"""One tls_factor_precond at n = PROF_N (m = 8n) for an ncu launch list of the Cholesky kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_19028_b200 import tlsrqi
n = int(os.environ.get("PROF_N", 2000)); m = 8 * n
A = torch.randn((m, n), dtype=torch.float64, device="cuda")
M = tlsrqi.matrix(A); ws = tlsrqi.workspace(M)
rc, R, fi = tlsrqi.tls_factor_precond(M, "fp16", ws=ws)
torch.cuda.synchronize(); print("ok", rc)
