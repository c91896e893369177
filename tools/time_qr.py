"""Device time of the Householder-QR preconditioner (tls_factor_precond_qr, NEXT-2) next to the
Gram-Cholesky one (tls_factor_precond) on the same A, CUDA events around each call; and the
agreement of the two R~ with each other (both approximate the same R of A D^{-1})."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2305_19028_b200 import tlsrqi

shapes = [(4096, 512), (16384, 1024), (65536, 2048)] if len(sys.argv) < 2 else \
    [tuple(int(v) for v in s.split("x")) for s in sys.argv[1:]]
for m, n in shapes:
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g) * \
        torch.logspace(0, -2, n, dtype=torch.float64, device="cuda")[None, :]
    M = tlsrqi.matrix(A)
    for fmt in ("fp16", "bf16"):
        wq = torch.empty(int(tlsrqi.lib().tls_qr_workspace_size(M, tlsrqi.PREC[fmt], 1)), dtype=torch.uint8, device="cuda")
        wc = tlsrqi.workspace(M)
        out = {}
        for name, fn in (("qr", lambda: tlsrqi.tls_factor_precond_qr(M, fmt, ws=wq)),
                         ("chol", lambda: tlsrqi.tls_factor_precond(M, fmt, ws=wc))):
            rc, R, fi = fn()
            assert rc == 0, (name, rc)
            ts = []
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                rc, R, fi = fn()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            out[name] = (min(ts), fi["launches"], tlsrqi.tls_precond_export(R)[0])
        dq = out["qr"][2]
        dc = out["chol"][2]
        rel = np.linalg.norm(np.abs(dq) - np.abs(dc)) / np.linalg.norm(dc)
        print(f"{m}x{n} {fmt}: qr {out['qr'][0]:.3f} ms ({out['qr'][1]} launches)  chol {out['chol'][0]:.3f} ms"
              f"  ||R_qr - R_chol||/||R_chol|| = {rel:.2e}", flush=True)
