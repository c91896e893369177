"""Device time of the dense passes (tls_pass includes the fixed-order reduce; both timed)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_19028_b200 import tlsrqi
for m, n in ((1 << 20, 1024), (1 << 16, 2048), (1 << 19, 512)):
    A = torch.randn((m, n), dtype=torch.float64, device="cuda")
    M = tlsrqi.matrix(A); ws = tlsrqi.workspace(M)
    q = torch.randn((2, n), dtype=torch.float64, device="cuda")
    b = torch.randn(m, dtype=torch.float64, device="cuda")
    for name, args in (("op2", (0, q, None)), ("op1", (0, q[:1], None)), ("resid", (1, q[0], b))):
        tlsrqi.tls_pass(M, args[0], args[1], args[2], ws=ws)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(30):
            tlsrqi.tls_pass(M, args[0], args[1], args[2], ws=ws)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 30
        print(f"m={m} n={n} {name:5s}: {ms:.3f} ms  {8 * m * n / ms / 1e9:7.2f} TB/s (incl. reduce + copy-out)", flush=True)
    del A, M, ws
    torch.cuda.empty_cache()
