"""The split-role fused Gram (k_gram_fused2, opt-in TLS_GRAM_FUSED=2, n > 896, K_t = 64) against the
two-kernel path (k_round_scaled + k_gram_tc2, TLS_GRAM_FUSED=0): G bit-identical when both use
the same split count (TLS_GRAM_NSPLIT) and one segment (TLS_GRAM_SEGS=1), and device time of tls_gram (CUDA events, median of 5)
of each path as it runs by default.

  python tools/time_gram_fused2.py
"""
import os
import statistics
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(m, n, fmt, tag, odd):
    import numpy as np
    import torch
    from paper_2305_19028_b200 import tlsrqi
    torch.manual_seed(0)
    A = torch.randn((m, n + odd), dtype=torch.float64, device="cuda")
    M = tlsrqi.matrix(A, n=n) if odd else tlsrqi.matrix(A)
    ws = tlsrqi.workspace(M)
    d = torch.exp2(torch.randint(-3, 4, (n,), device="cuda").double())
    rc, G = tlsrqi.tls_gram(M, fmt, d, 64, ws=ws)
    ts = []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        tlsrqi.tls_gram(M, fmt, d, 64, ws=ws)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    np.save(f"/tmp/Gf2_{tag}_{m}_{n}_{fmt}.npy", G.cpu().numpy())
    return rc, statistics.median(ts)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        m, n, fmt, tag, odd = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5], int(sys.argv[6])
        rc, ms = run(m, n, fmt, tag, odd)
        print(f"{rc} {ms:.3f}")
        sys.exit(0)
    import numpy as np
    shapes = [(1 << 20, 1024, "fp16", 0), (1 << 20, 1024, "bf16", 0), (300001, 1000, "fp16", 2), (65536, 2048, "fp16", 0),
              (200000, 2000, "bf16", 0), (9000, 1100, "fp16", 0)]
    for m, n, fmt, odd in shapes:
        res = {}
        for tag, env in (("fused2", {"TLS_GRAM_FUSED": "2"}), ("twokernel", {"TLS_GRAM_FUSED": "0"}),
                         ("fused2_s3", {"TLS_GRAM_FUSED": "2", "TLS_GRAM_NSPLIT": "3"}),
                         ("twokernel_s3", {"TLS_GRAM_FUSED": "0", "TLS_GRAM_NSPLIT": "3", "TLS_GRAM_SEGS": "1"})):
            out = subprocess.run([sys.executable, __file__, "--one", str(m), str(n), fmt, tag, str(odd)],
                                 env=dict(os.environ, **env), capture_output=True, text=True)
            res[tag] = out.stdout.strip() or out.stderr[-600:]
        line = f"{m}x{n} {fmt}: fused2 {res['fused2']} ms | two-kernel {res['twokernel']} ms"
        try:
            a = np.load(f"/tmp/Gf2_fused2_s3_{m}_{n}_{fmt}.npy")
            b = np.load(f"/tmp/Gf2_twokernel_s3_{m}_{n}_{fmt}.npy")
            c = np.load(f"/tmp/Gf2_fused2_{m}_{n}_{fmt}.npy")
            d = np.load(f"/tmp/Gf2_twokernel_{m}_{n}_{fmt}.npy")
            line += (f" | 3 splits each: bit-identical {np.array_equal(a, b)} | defaults: max|diff|/max|G| "
                     f"{np.abs(c - d).max() / np.abs(d).max():.2e}")
        except Exception as e:  # noqa: BLE001
            line += f" | compare failed: {e}"
        print(line, flush=True)
