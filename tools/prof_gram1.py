"""One tls_gram call at cfg4w size (for an ncu launch list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import tlsgen
from paper_2305_19028_b200 import tlsrqi
P = tlsgen.dense_problem(1 << 20, 1024, 1e4, 1e-3, 4, twin=True, device="cuda", keep_factors=False)
M = tlsrqi.matrix(P.A)
ws = tlsrqi.workspace(M)
d = torch.ones(1024, dtype=torch.float64, device="cuda")
for _ in range(2):
    tlsrqi.tls_gram(M, "fp16", d, int(os.environ.get("KT", 64)), ws=ws)
torch.cuda.synchronize()
