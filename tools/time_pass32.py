"""Device time of the 2-RHS operator pass: fp64 k_pass vs the u_p = fp32 k_pass32
(R23), on a dense m x n A (default the cfg4w shape), per-kernel times from the
library's event profiler.  python tools/time_pass32.py [m] [n] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_19028_b200 import tlsrqi as T

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g)
q = torch.randn((2, n), dtype=torch.float64, device="cuda", generator=g)
M = T.matrix(A)
ws = T.workspace(M)
R = T.tls_precond_import(torch.eye(n, dtype=torch.float64).numpy(), torch.ones(n, dtype=torch.float64).numpy(),
                         1.0, "fp64")
T.tls_pass(M, 0, q, ws=ws)
T.tls_pass_fp32(M, R, q, ws=ws)
torch.cuda.synchronize()
T.tls_profile_enable(1)
for _ in range(reps):
    T.tls_pass(M, 0, q, ws=ws)
    T.tls_pass_fp32(M, R, q, ws=ws)
torch.cuda.synchronize()
p = T.tls_profile_read()
t64 = p["pass_op2"]["ms"] / p["pass_op2"]["count"]
t32 = p["pass_op2_fp32"]["ms"] / p["pass_op2_fp32"]["count"]
print(f"m={m} n={n}: fp64 op pass {t64:.3f} ms ({8*m*n/t64/1e9:.2f} TB/s)   "
      f"fp32 op pass {t32:.3f} ms ({4*m*n/t32/1e9:.2f} TB/s)   ratio {t64/t32:.2f}")
