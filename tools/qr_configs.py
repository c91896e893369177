"""The BASELINE dense configs with both preconditioners through the GPU path (NEXT-2): the
Gram-Cholesky R~ (tls_factor_precond) and the Householder-QR R~ in u_f
(tls_factor_precond_qr), each followed by the same tls_rqi_pcgtls.  Per run: factor time,
solve time (CUDA events, best of --reps), status, RQI steps, CGLS bootstrap iterations and
total PCG iterations.  JSON lines to stdout.  cfg3 (CSR) has no QR path."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import tlsgen
from paper_2305_19028_b200 import tlsrqi as T


def timed(fn, reps):
    best, out = None, None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return best, out


ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--configs", default="cfg1,cfg2w,cfg5:k1e2:e1e-3,cfg5:k1e4:e1e-6,cfg4w")
args = ap.parse_args()
for name in args.configs.split(","):
    dev = "cuda" if name.startswith(("cfg4", "cfg5")) else "cpu"
    P = tlsgen.config(name, device=dev, keep_factors=False) if dev == "cuda" else tlsgen.config(name)
    A = P.A if torch.is_tensor(P.A) else torch.as_tensor(np.ascontiguousarray(P.A), device="cuda")
    b = P.b if torch.is_tensor(P.b) else torch.as_tensor(P.b, device="cuda")
    M = T.matrix(T.dense_operand(A), n=A.shape[1])
    ws = T.workspace(M)
    for u_f in ("fp16", "bf16"):
        qws = torch.empty(int(T.lib().tls_qr_workspace_size(M, T.PREC[u_f], 1)), dtype=torch.uint8, device="cuda")
        for kind, fac in (("cholesky", lambda: T.tls_factor_precond(M, u_f, ws=ws)),
                          ("qr", lambda: T.tls_factor_precond_qr(M, u_f, ws=qws))):
            t_f, (rc, R, fi) = timed(fac, args.reps)
            rec = {"config": name, "u_f": u_f, "precond": kind, "factor_ms": round(t_f, 3), "factor_status": rc,
                   "pivot": fi["chol_pivot"]}
            if rc == 0:
                t_s, (rc2, x, sig, info) = timed(lambda: T.tls_rqi_pcgtls(M, b, R, ws=ws), args.reps)
                rec.update({"solve_ms": round(t_s, 3), "status": info["status_name"], "rqi": info["rqi_iters"],
                            "boot": info["boot_iters"], "pcg_total": sum(p[0] + p[1] for p in info["pcg_iters"]),
                            "sigma": sig})
            print(json.dumps(rec), flush=True)
        del qws
    del P, A, b, M, ws
    torch.cuda.empty_cache()
