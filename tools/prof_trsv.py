"""A few tls_precond_apply launches (fp16, n from env) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2305_19028_b200 import tlsrqi
n = int(os.environ.get("PROF_N", 1024)); fmt = os.environ.get("PROF_FMT", "fp16")
rng = np.random.default_rng(0)
R = np.triu(rng.standard_normal((n, n))) / n
R[np.diag_indices(n)] = 1.0 + rng.random(n)
R = R.astype(np.float16).astype(np.float64)
pc = tlsrqi.tls_precond_import(R, np.ones(n), 1.0, fmt)
Y = torch.randn((2, n), dtype=torch.float64, device="cuda")
for _ in range(3):
    tlsrqi.tls_precond_apply(pc, 0, Y)
torch.cuda.synchronize(); print("ok")
