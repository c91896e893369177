"""Accuracy and time of the tensor-core Gram variants at full cfg4w size (2^20 x 1024,
u_f fp16): error against the fp64 Gram of the same rounded A^ (relative to |A^|^T|A^|),
smallest eigenvalue, device time.  Variants via TLS_GRAM_SUPER / TLS_GRAM_KAHAN (read
by the library at each launch).  Also runs the whole solve for each variant so the
RQI/PCG counts can be compared."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import tlsgen
from paper_2305_19028_b200 import tlsrqi

m = int(os.environ.get("GC_M", 1 << 20)); n = int(os.environ.get("GC_N", 1024))
kappa = float(os.environ.get("GC_KAPPA", 1e4))
P = tlsgen.dense_problem(m, n, kappa, 1e-3, 4, twin=True, device="cuda", keep_factors=False)
M = tlsrqi.matrix(P.A)
ws = tlsrqi.workspace(M)
colmax, sumsq = tlsrqi.tls_colstats(M, ws=ws)
e = torch.frexp(colmax)[1]
d = torch.ldexp(torch.ones_like(colmax), e - 1)
Ah = (P.A / d).to(torch.float16).to(torch.float64)   # fp64 -> fp16 is RNE (direct)
G64 = (Ah.T @ Ah).cpu().numpy()
absG = (Ah.abs().T @ Ah.abs()).cpu().numpy()
del Ah
torch.cuda.empty_cache()
L64 = np.linalg.eigvalsh(G64)
print(f"fp64 Gram of A^: lam_min {L64[0]:.4e} lam_max {L64[-1]:.4e}", flush=True)
variants = [(v.split(":")[0], v.split(":")[1], v.split(":")[2]) for v in
            os.environ.get("GC_VARIANTS", "64:16:0,64:64:0,64:256:0,64:1024:0,64:4096:0,64:64:1").split(",")]
for K_t, sup, kah in variants:
    os.environ["TLS_GRAM_SUPER"] = sup
    os.environ["TLS_GRAM_KAHAN"] = kah
    rc, G = tlsrqi.tls_gram(M, "fp16", d, int(K_t), ws=ws)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        tlsrqi.tls_gram(M, "fp16", d, int(K_t), ws=ws)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    Gn = G.cpu().numpy()
    err = np.abs(Gn - G64) / absG
    L = np.linalg.eigvalsh(Gn)
    o = tlsrqi.tls_rqi_opts_default(gram_chunk=int(K_t))
    rcf, R, fi = tlsrqi.tls_factor_precond(M, "fp16", opts=o, ws=ws)
    line = (f"K_t={K_t:>4} super={sup:>3} kahan={kah}: {ms:7.2f} ms (tls_gram incl. rounding pass)  "
            f"max rel err {err.max():.2e} median {np.median(err):.2e}  lam_min {L[0]:.4e}")
    if R is not None:
        rc2, x, sig, info = tlsrqi.tls_rqi_pcgtls(M, P.b, R, ws=ws)
        line += f"  solve {info['status_name']} K={info['rqi_iters']} B0={info['boot_iters']} pcg={info['pcg_iters']}"
    else:
        line += f"  factor {fi['status_name']} pivot {fi['chol_pivot']}"
    print(line, flush=True)
