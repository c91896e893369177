"""Profiling driver for the preconditioner build on a cfg4-sized operand:
tls_factor_precond (colstats pass, Gram pre-pass + tcgen05 SYRK + reduce,
Cholesky, packing) a few times.  Used under ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_19028_b200 import tlsrqi

m = int(os.environ.get("PROF_M", 1 << 20)); n = int(os.environ.get("PROF_N", 1024))
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn((m, n), generator=g, dtype=torch.float64, device="cuda")
M = tlsrqi.matrix(A)
ws = tlsrqi.workspace(M)
for _ in range(int(os.environ.get("PROF_REPS", 2))):
    rc, R, info = tlsrqi.tls_factor_precond(M, os.environ.get("PROF_UF", "fp16"), ws=ws)
torch.cuda.synchronize()
print("ok", rc)
