"""The Gram's rounding pass fl_uf(A D^-1) in its forms (TLS_ROUND=1: one row in flight per
thread, round 2's kernel; 2: two rows, the default; a cp.async-staged form, measured in
profiles/r02f_round.log, was removed as slower), alone
(TLS_GRAM_SEGS=1) and overlapped with the segmented tcgen05 SYRK (8 / 16 segments): device time of
tls_gram (CUDA events, median of 5) and G bit-identical across the forms with the same segments.

  python tools/time_round.py
"""
import os
import statistics
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(m, n, fmt, tag):
    import numpy as np
    import torch
    from paper_2305_19028_b200 import tlsrqi
    torch.manual_seed(0)
    A = tlsrqi.dense_operand(torch.randn((m, n), dtype=torch.float64, device="cuda"))
    M = tlsrqi.matrix(A)
    ws = tlsrqi.workspace(M)
    d = torch.ones(n, dtype=torch.float64, device="cuda") * 8
    rc, G = tlsrqi.tls_gram(M, fmt, d, 64, ws=ws)
    ts = []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        tlsrqi.tls_gram(M, fmt, d, 64, ws=ws)
        e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    np.save(f"/tmp/Gr_{tag}.npy", G.cpu().numpy())
    return rc, statistics.median(ts)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        m, n, fmt, tag = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
        rc, ms = run(m, n, fmt, tag)
        print(f"{rc} {ms:.4f}")
        sys.exit(0)
    import numpy as np
    shapes = [(1 << 20, 1024, "fp16"), (1 << 20, 1024, "bf16"), (65536, 2048, "fp16"), (200000, 2000, "fp16"),
              (70001, 257, "fp16")]
    for m, n, fmt in shapes:
        for segs in ("1", "8", "16"):
            line, base = [], None
            for rv in ("1", "2"):
                tag = f"{m}_{n}_{fmt}_{segs}_{rv}"
                out = subprocess.run([sys.executable, __file__, "--one", str(m), str(n), fmt, tag],
                                     env=dict(os.environ, TLS_ROUND=rv, TLS_GRAM_SEGS=segs), capture_output=True,
                                     text=True, timeout=600)
                res = out.stdout.strip() or out.stderr[-400:]
                try:
                    g = np.load(f"/tmp/Gr_{tag}.npy")
                    if base is None:
                        base = g
                    same = bool(np.array_equal(g, base))
                except FileNotFoundError:
                    same = None
                line.append(f"round={rv}: {res} ms same-G={same}")
            print(f"{m}x{n} {fmt} segs={segs}: " + " | ".join(line), flush=True)
