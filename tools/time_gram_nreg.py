"""tls_gram time (CUDA events, median of 7) and a SHA-256 of G for the build that is loaded:
used to A/B the compile-time register cap of k_gram_tc2 (TLS_EXTRA_NVCC=-DTLS_T2_MAXNREG=128).

  python tools/time_gram_nreg.py <tag>
"""
import hashlib
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2305_19028_b200 import tlsrqi  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "default"
for m, n in ((1 << 20, 1024), (65536, 2048), (200000, 2000)):
    for fmt in ("fp16", "bf16"):
        torch.manual_seed(0)
        A = torch.randn((m, n), dtype=torch.float64, device="cuda")
        M = tlsrqi.matrix(A)
        ws = tlsrqi.workspace(M)
        d = torch.ones(n, dtype=torch.float64, device="cuda") * 8
        rc, G = tlsrqi.tls_gram(M, fmt, d, 64, ws=ws)
        ts = []
        for _ in range(7):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            tlsrqi.tls_gram(M, fmt, d, 64, ws=ws)
            e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        h = hashlib.sha256(G.cpu().numpy().tobytes()).hexdigest()[:16]
        print(f"{tag}: {m}x{n} {fmt}: rc={rc} {statistics.median(ts):.4f} ms (min {min(ts):.4f}) G sha {h}", flush=True)
        del A, M, ws, G
