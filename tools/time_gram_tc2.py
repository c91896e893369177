"""The 128 x 256-block Gram (k_gram_tc2, UMMA N = 256, default) against the 128 x 128-tile kernel
(k_gram_tc, TLS_GRAM_TC=128): device time of tls_gram (CUDA events, median of 5) and the
difference of the two G's (the chunk sums are the same; the split boundaries differ, so the fp64
sums of the split partials are grouped differently).

  python tools/time_gram_tc2.py
"""
import os
import statistics
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(m, n, fmt, K_t, tag):
    import numpy as np
    import torch
    from paper_2305_19028_b200 import tlsrqi
    torch.manual_seed(0)
    A = torch.randn((m, n), dtype=torch.float64, device="cuda")
    M = tlsrqi.matrix(A)
    ws = tlsrqi.workspace(M)
    d = torch.ones(n, dtype=torch.float64, device="cuda") * 8
    rc, G = tlsrqi.tls_gram(M, fmt, d, K_t, ws=ws)
    ts = []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        tlsrqi.tls_gram(M, fmt, d, K_t, ws=ws)
        e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    np.save(f"/tmp/G_{tag}_{m}_{n}_{fmt}_{K_t}.npy", G.cpu().numpy())
    return rc, statistics.median(ts)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        m, n, fmt, K_t, tag = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5]), sys.argv[6]
        rc, ms = run(m, n, fmt, K_t, tag)
        print(f"{rc} {ms}")
        sys.exit(0)
    import numpy as np
    shapes = [(1 << 20, 1024, "fp16", 64), (1 << 20, 1024, "bf16", 64), (65536, 2048, "fp16", 64),
              (200000, 2000, "fp16", 64), (70001, 256, "fp16", 64), (5000, 64, "bf16", 64), (2100, 514, "fp16", 64),
              (3000, 300, "fp16", 2048), (1 << 20, 1024, "fp16", 8192)]
    for m, n, fmt, K_t in shapes:
        res = {}
        for tag, env in (("tc2", {"TLS_GRAM_TC": "256"}), ("tc128", {"TLS_GRAM_TC": "128"})):
            out = subprocess.run([sys.executable, __file__, "--one", str(m), str(n), fmt, str(K_t), tag],
                                 env=dict(os.environ, **env), capture_output=True, text=True)
            res[tag] = out.stdout.strip() or out.stderr[-800:]
        line = f"{m}x{n} {fmt} K_t={K_t}: tc2 {res['tc2']} ms | tc128 {res['tc128']} ms"
        try:
            a = np.load(f"/tmp/G_tc2_{m}_{n}_{fmt}_{K_t}.npy")
            b = np.load(f"/tmp/G_tc128_{m}_{n}_{fmt}_{K_t}.npy")
            line += (f" | identical {np.mean(a == b):.4f} max|diff|/max|G| {np.abs(a - b).max() / np.abs(b).max():.2e}"
                     f" symmetric {np.array_equal(a, a.T)}")
        except Exception as e:  # noqa: BLE001
            line += f" | compare failed: {e}"
        print(line, flush=True)
