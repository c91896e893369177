"""Profiling driver: the fp64 Gram (k_gram_f64, DMMA) at cfg5 size.  Used under ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_19028_b200 import tlsrqi
A = torch.randn((65536, 2048), dtype=torch.float64, device="cuda")
M = tlsrqi.matrix(A); ws = tlsrqi.workspace(M)
d = torch.ones(2048, dtype=torch.float64, device="cuda")
for _ in range(2):
    tlsrqi.tls_gram(M, "fp64", d, 64, ws=ws)
torch.cuda.synchronize()
