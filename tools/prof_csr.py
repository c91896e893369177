"""Profiling driver: CSR operator passes (k_csr_rows + k_csr_cols, 2 RHS) on cfg3 through
the C ABI.  Used under ncu only."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import tlsgen
from paper_2305_19028_b200 import tlsrqi
P = tlsgen.config("cfg3")
M = tlsrqi.matrix_csr(torch.as_tensor(P.rowptr, device="cuda"), torch.as_tensor(P.colidx, device="cuda"),
                      torch.as_tensor(P.vals, device="cuda"), P.n)
ws = tlsrqi.workspace(M)
q = torch.randn((2, P.n), dtype=torch.float64, device="cuda")
for _ in range(4):
    tlsrqi.tls_pass(M, 0, q, ws=ws)
torch.cuda.synchronize()
