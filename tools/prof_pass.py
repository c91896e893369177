"""Profiling driver: a few launches of the dominant kernel (operator pass, 2 RHS) on a
cfg4-sized operand (2^20 x 1024 fp64) through the C ABI.  Used under ncu only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2305_19028_b200 import tlsrqi

m = int(os.environ.get("PROF_M", 1 << 20))
n = int(os.environ.get("PROF_N", 1024))
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn((m, n), generator=g, dtype=torch.float64, device="cuda")
M = tlsrqi.matrix(A)
ws = tlsrqi.workspace(M)
q = torch.randn((2, n), generator=g, dtype=torch.float64, device="cuda")
for _ in range(int(os.environ.get("PROF_REPS", 4))):
    v, s = tlsrqi.tls_pass(M, 0, q, ws=ws)
torch.cuda.synchronize()
print("ok", float(s[0]))
