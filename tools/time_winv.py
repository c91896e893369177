"""PCG step (a6 + a8) and solve time with the preconditioner applied by substitution
(precond_apply = 1) or through the explicit inverse W (= 2, R24), per n; plus the one-off
cost of forming W.  python tools/time_winv.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import tlsgen
from paper_2305_19028_b200 import tlsrqi as T

for n in (1024, 2000, 2048):
    P = tlsgen.dense_problem(16 * n, n, 1e3, 1e-3, 7, twin=True, device="cuda", keep_factors=False)
    M = T.matrix(P.A)
    ws = T.workspace(M)
    rc, R, _ = T.tls_factor_precond(M, "fp16", ws=ws)
    out = []
    for mode in (1, 2):
        o = T.tls_rqi_opts_default(precond_apply=mode)
        T.tls_rqi_pcgtls(M, P.b, R, ws=ws, opts=o)       # warm-up (forms W once for mode 2)
        torch.cuda.synchronize()
        T.tls_profile_enable(1)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            rc, x, sig, info = T.tls_rqi_pcgtls(M, P.b, R, ws=ws, opts=o)
        e1.record(); torch.cuda.synchronize()
        p = T.tls_profile_read()
        T.tls_profile_enable(0)
        st = p["pcg_step"]["ms"] / max(1, p["pcg_step"]["count"])
        out.append(f"mode {mode}: solve {e0.elapsed_time(e1) / 5:.3f} ms, pcg_step {st * 1e3:.1f} us "
                   f"(K={info['rqi_iters']} B0={info['boot_iters']})")
    # the one-off W
    rc, R2, _ = T.tls_factor_precond(M, "fp16", ws=ws)
    Y = torch.zeros((1, n), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    T.tls_precond_apply(R2, 2, Y)
    e1.record(); torch.cuda.synchronize()
    print(f"n={n}: " + " | ".join(out) + f" | forming W + one apply {e0.elapsed_time(e1):.3f} ms", flush=True)
