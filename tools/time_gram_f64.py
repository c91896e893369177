"""tls_gram for u_f fp32 / fp64 (fp64-accumulating CUDA-core kernel) at cfg5 size."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_19028_b200 import tlsrqi
m, n = 65536, 2048
A = torch.randn((m, n), dtype=torch.float64, device="cuda")
M = tlsrqi.matrix(A); ws = tlsrqi.workspace(M)
d = torch.ones(n, dtype=torch.float64, device="cuda") * 8
for fmt in ("fp32", "fp64"):
    rc, G = tlsrqi.tls_gram(M, fmt, d, 64, ws=ws)
    ref = (A / d).to(torch.float32).double() if fmt == "fp32" else A / d
    Gr = ref.T @ ref
    err = float(((G - Gr).abs() / (ref.abs().T @ ref.abs())).max())
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        tlsrqi.tls_gram(M, fmt, d, 64, ws=ws)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{fmt}: {ms:.2f} ms  {m * n * (n + 128) / ms / 1e9:.1f} TFLOP/s over the SYRK tiles  max rel err {err:.2e}", flush=True)
