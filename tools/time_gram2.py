"""Device time of k_gram_tc variants (env TLS_GRAM_*), cfg4w size, via tls_gram (warm, events)."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_19028_b200 import tlsrqi
m, n = 1 << 20, 1024
A = torch.randn((m, n), dtype=torch.float64, device="cuda")
M = tlsrqi.matrix(A)
ws = tlsrqi.workspace(M)
d = torch.ones(n, dtype=torch.float64, device="cuda") * 8
for epi in ("2",):
    for sup in ("16", "32", "64"):
        os.environ["TLS_GRAM_EPI"] = epi
        os.environ["TLS_GRAM_SUPER"] = sup
        for K_t in (64, 8192):
            tlsrqi.tls_gram(M, "fp16", d, K_t, ws=ws)
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                tlsrqi.tls_gram(M, "fp16", d, K_t, ws=ws)
            e1.record(); torch.cuda.synchronize()
            print(f"epi={epi} super={sup} K_t={K_t:5d}: {e0.elapsed_time(e1) / 3:7.3f} ms", flush=True)
