"""The fused Gram (k_gram_fused: rounding inside the tcgen05 kernel, A^ in an L2 ring) against the
two-kernel path (k_round_scaled + k_gram_tc, TLS_GRAM_FUSED=0): bit-identical G, and device time
of tls_gram (CUDA events, median of 5) at the bench shape and cfg5's.

  python tools/time_gram_fused.py [m x n ...]
"""
import os
import statistics
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(m, n, fmt, K_t):
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
    g = G.cpu().numpy()
    np.save(f"/tmp/G_{os.environ.get('TLS_GRAM_FUSED', '1')}_{m}_{n}_{fmt}.npy", g)
    return rc, statistics.median(ts)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        m, n, fmt, K_t = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5])
        rc, ms = run(m, n, fmt, K_t)
        print(f"{rc} {ms}")
        sys.exit(0)
    import numpy as np
    shapes = [(1 << 20, 1024, "fp16"), (65536, 2048, "fp16"), (1 << 20, 1024, "bf16"), (70001, 256, "fp16"),
              (5000, 64, "bf16"), (2100, 514, "fp16")]
    for m, n, fmt in shapes:
        res = {}
        for fused in ("1", "0"):             # TLS_GRAM_FUSED=1: the fused kernel (opt-in)
            out = subprocess.run([sys.executable, __file__, "--one", str(m), str(n), fmt, "64"],
                                 env=dict(os.environ, TLS_GRAM_FUSED=fused), capture_output=True, text=True,
                                 timeout=600)
            res[fused] = out.stdout.strip() or out.stderr[-800:]
        try:
            g1 = np.load(f"/tmp/G_1_{m}_{n}_{fmt}.npy")
            g0 = np.load(f"/tmp/G_0_{m}_{n}_{fmt}.npy")
        except FileNotFoundError:
            print(f"{m}x{n} {fmt}: fused {res['1']} | two-kernel {res['0']}", flush=True)
            continue
        print(f"{m}x{n} {fmt}: fused {res['1']} | two-kernel {res['0']} | bit-identical {np.array_equal(g1, g0)} "
              f"max|diff| {np.max(np.abs(g1 - g0)):.3e}", flush=True)
