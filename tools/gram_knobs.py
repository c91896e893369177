"""Where the tensor-core Gram's time goes: tls_gram on 2^20 x 1024 fp16 with the epilogue
knob TLS_GRAM_EPI (0: no TMEM drain, 1: TMEM loads only, 2: full) and K_t in {64, 8192}
(diagnostics; EPI < 2 gives a wrong G).  Per-call device time from the profiler."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_19028_b200 import tlsrqi
n = 1024; m = 1 << 20
A = torch.randn((m, n), dtype=torch.float64, device="cuda")
M = tlsrqi.matrix(A); ws = tlsrqi.workspace(M)
d = torch.ones(n, dtype=torch.float64, device="cuda") * 8
for epi in ("2", "1", "0"):
    for K_t in (64, 8192):
        os.environ["TLS_GRAM_EPI"] = epi
        tlsrqi.tls_gram(M, "fp16", d, K_t, ws=ws)
        tlsrqi.tls_profile_enable(1)
        for _ in range(5):
            tlsrqi.tls_gram(M, "fp16", d, K_t, ws=ws)
        p = tlsrqi.tls_profile_read()
        tlsrqi.tls_profile_enable(0)
        print(f"EPI={epi} K_t={K_t}: tls_gram {p['gram']['ms'] / p['gram']['count']:.3f} ms", flush=True)
