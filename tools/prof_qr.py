"""One tls_factor_precond_qr (NEXT-2) on an m x n Gaussian A for ncu (default 65536 x 2048, fp16)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_19028_b200 import tlsrqi

m = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
fmt = sys.argv[3] if len(sys.argv) > 3 else "fp16"
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
M = tlsrqi.matrix(A)
rc, R, info = tlsrqi.tls_factor_precond_qr(M, fmt)
torch.cuda.synchronize()
print("rc", rc, "launches", info["launches"])
