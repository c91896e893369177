"""Non-pass time of one PCG iteration (NEXT-3): a solve on a SHORT A (m = 8192 rows, n = 1024,
so the operator pass is ~10 us) with budget_rule = until tol and a loose tol, timed with CUDA
events around the whole PCG loop; per iteration = loop time / iterations, minus the pass
kernel's own event-timed duration.  Compares the substitution step (k_pcg_step, 8-CTA
clusters), the explicit-inverse step with the separate reduction (TLS_FUSE_REDUCE=0) and the
fused step (reduction folded into k_wpcg_step_coop).

  python tools/time_pcg_iter.py [--n 1024] [--m 8192]
"""
import argparse
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def one(mode, m, n):
    import numpy as np
    import torch
    import tlsgen
    from paper_2305_19028_b200 import tlsrqi as T
    torch.cuda.set_device(0)
    P = tlsgen.dense_problem(m, n, 1e2, 1e-3, 3, twin=True, device="cuda", keep_factors=False)
    M = T.matrix(P.A)
    ws = T.workspace(M)
    rc, R, _ = T.tls_factor_precond(M, "fp16", ws=ws)
    pa = 1 if mode == "subst" else 2
    o = T.tls_rqi_opts_default(precond_apply=pa, boot_max=400, boot_tol=1e-300)   # bootstrap = 400 iterations
    o.max_outer = 1
    for _ in range(2):
        T.tls_rqi_pcgtls(M, P.b, R, opts=o, ws=ws)
    torch.cuda.synchronize()
    # (a) per-kernel event timing (profiling on: the host loop, no graph)
    T.tls_profile_enable(True)
    rc, x, sig, info = T.tls_rqi_pcgtls(M, P.b, R, opts=o, ws=ws)
    torch.cuda.synchronize()
    prof = T.tls_profile_read()
    T.tls_profile_enable(False)
    # (b) the whole solve without profiling (the graph-captured loop unless TLS_PCG_GRAPH=0)
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc, x, sig, info = T.tls_rqi_pcgtls(M, P.b, R, opts=o, ws=ws)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    total_ms = min(ts)
    it = info["boot_iters"]
    pass_us = 1e3 * prof["pass_op2"]["ms"] / max(1, prof["pass_op2"]["count"])
    per_iter = 1e3 * total_ms / max(1, it)
    return {"mode": mode, "graph": os.environ.get("TLS_PCG_GRAPH", "1") != "0", "pdl": os.environ.get("TLS_PDL", "1") != "0",
            "wstep_ctas": os.environ.get("TLS_WSTEP_CTAS", "auto"),
            "m": m, "n": n, "boot_iters": it,
            "solve_ms": total_ms, "launches": info["launches"], "pass_us_per_iter": pass_us,
            "step_us_per_iter": 1e3 * prof["pcg_step"]["ms"] / max(1, prof["pcg_step"]["count"]),
            "reduce_us_per_iter": 1e3 * prof["reduce"]["ms"] / max(1, prof["reduce"]["count"]),
            "per_iter_us": per_iter, "non_pass_us_per_iter": per_iter - pass_us}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--m", type=int, default=8192)
    ap.add_argument("--mode", default="")
    args = ap.parse_args()
    if args.mode:
        print(json.dumps(one(args.mode, args.m, args.n)))
        return
    for mode, env in (("subst", {"TLS_PCG_GRAPH": "0", "TLS_PDL": "0"}), ("subst", {"TLS_PDL": "0"}), ("subst", {}),
                      ("subst", {"TLS_FUSE_REDUCE": "0"}),
                      ("winv_sep", {"TLS_FUSE_REDUCE": "0", "TLS_PCG_GRAPH": "0", "TLS_PDL": "0"}),
                      ("winv_fused", {"TLS_PCG_GRAPH": "0", "TLS_PDL": "0"}), ("winv_fused", {"TLS_PDL": "0"}),
                      ("winv_fused", {}), ("winv_fused", {"TLS_WSTEP_CTAS": "64"}), ("winv_fused", {"TLS_WSTEP_CTAS": "32"})):
        e = dict(os.environ, **env)
        out = subprocess.run([sys.executable, __file__, "--mode", mode, "--m", str(args.m), "--n", str(args.n)],
                             env=e, capture_output=True, text=True)
        print(out.stdout.strip() or out.stderr[-2000:], flush=True)


if __name__ == "__main__":
    main()
