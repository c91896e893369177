"""Device time of tls_gram (rounding pass + tcgen05 SYRK + reduce) for several m and K_t."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_19028_b200 import tlsrqi
n = int(os.environ.get("TG_N", 1024))
for m in (1 << 16, 1 << 18, 1 << 20):
    A = torch.randn((m, n), dtype=torch.float64, device="cuda")
    M = tlsrqi.matrix(A)
    ws = tlsrqi.workspace(M)
    d = torch.ones(n, dtype=torch.float64, device="cuda") * 8
    for K_t in (64, 256, 1024, 8192):
        tlsrqi.tls_gram(M, "fp16", d, K_t, ws=ws)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            tlsrqi.tls_gram(M, "fp16", d, K_t, ws=ws)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        fl = m * n * (n + 128)  # upper 128-tiles incl. diagonal tiles
        print(f"m={m:8d} K_t={K_t:5d}: {ms:8.3f} ms  ({fl / ms / 1e9:7.1f} TFLOP/s over the SYRK tiles)", flush=True)
    del A, M, ws
    torch.cuda.empty_cache()
