"""Run the whole hot path (tls_factor_precond + tls_rqi_pcgtls) on every BASELINE.json
config on one GPU and report status, counts and time-to-solution (CUDA events,
median of REPS runs after one warm-up).  cfg5 is the full conditioning sweep:
kappa in {1e2,1e4,1e6,1e8} x eps in {1e-6,1e-3,1e-1} x u_f in {fp16,bf16,fp32} plus
the u_f = fp64 control, with the paper's u_f constraints (PAPER.md l.283-288 constr1
u_f <~ 1/kappa(A); l.366-391 constr2 on the shifted system) evaluated from the
construction (sigma'_n = s_n = 1/kappa) and the solve's sigma.

  python tools/run_configs.py [--only cfg1,cfg3,...] [--reps 3] [--out path]
"""
import argparse
import json
import math
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import tlsgen
from paper_2305_19028_b200 import tlsrqi as T

UROUND = {"fp16": 2.0 ** -11, "bf16": 2.0 ** -8, "fp32": 2.0 ** -24, "fp64": 2.0 ** -53}


EXTRA = {}   # --opts k=v,... applied to every solve (e.g. u_p=2,precond_apply=2)


def run(M, b, u_f, reps, ws, op_variant=0):
    opts = T.tls_rqi_opts_default(op_variant=op_variant, **EXTRA)
    def once():
        rc, R, fi = T.tls_factor_precond(M, u_f, ws=ws)
        if R is None:
            return rc, None, None, fi, None
        rc2, x, sig, info = T.tls_rqi_pcgtls(M, b, R, ws=ws, opts=opts)
        return rc2, x, sig, fi, info
    once()
    times = []
    out = None
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        out = once()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    rc, x, sig, fi, info = out
    rec = {"u_f": u_f, "op_variant": op_variant, "tts_s": statistics.median(times), "status": T.STATUS.get(rc, rc)}
    if info is None:
        rec.update({"chol_pivot": fi["chol_pivot"], "factor_status": fi["status_name"]})
        return rec, None
    rec.update({"termination": info["termination_name"], "rqi_iters": info["rqi_iters"],
                "boot_iters": info["boot_iters"], "pcg_iters": info["pcg_iters"], "sigma": sig,
                "passes": fi["passes"] + info["passes"], "launches": fi["launches"] + info["launches"]})
    return rec, x


def dense(P, u_f, reps, op_variant=0):
    A = P.A if torch.is_tensor(P.A) else torch.as_tensor(P.A)
    A = A.to("cuda")
    b = (P.b if torch.is_tensor(P.b) else torch.as_tensor(P.b)).to("cuda")
    M = T.matrix(A)
    ws = T.workspace(M)
    rec, x = run(M, b, u_f, reps, ws, op_variant)
    rec.update({"m": int(A.shape[0]), "n": int(A.shape[1])})
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/configs.json")
    ap.add_argument("--opts", default="", help="tls_rqi_opts_t overrides, e.g. u_p=2,precond_apply=2")
    args = ap.parse_args()
    for kv in filter(None, args.opts.split(",")):
        k, v = kv.split("=")
        EXTRA[k] = float(v) if "." in v or "e" in v else int(v)
    only = set(args.only.split(",")) if args.only else None
    res = {"gpu": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "opts": EXTRA, "runs": []}

    def want(k):
        return only is None or k in only

    for name in ("cfg1", "cfg2", "cfg2w", "cfg4", "cfg4w"):
        if not want(name):
            continue
        dev = "cuda" if name.startswith("cfg4") else "cpu"
        P = tlsgen.config(name, device=dev, keep_factors=False) if dev == "cuda" else tlsgen.config(name)
        for u_f in ([P.u_f, "bf16"] if name.startswith("cfg4") else [P.u_f]):
            rec = dense(P, u_f, args.reps)
            rec["config"] = name
            res["runs"].append(rec)
            print(json.dumps(rec), flush=True)
        if name in ("cfg1", "cfg2w", "cfg4w"):     # the paper's A-free operator
            rec = dense(P, P.u_f, args.reps, op_variant=1)
            rec["config"] = name
            res["runs"].append(rec)
            print(json.dumps(rec), flush=True)
        del P
        torch.cuda.empty_cache()
    if want("cfg3"):
        P = tlsgen.config("cfg3")
        M = T.matrix_csr(torch.as_tensor(P.rowptr, device="cuda"), torch.as_tensor(P.colidx, device="cuda"),
                         torch.as_tensor(P.vals, device="cuda"), P.n)
        ws = T.workspace(M)
        rec, _ = run(M, torch.as_tensor(P.b, device="cuda"), "fp16", args.reps, ws)
        rec.update({"config": "cfg3", "m": P.m, "n": P.n, "nnz": int(P.vals.size)})
        res["runs"].append(rec)
        print(json.dumps(rec), flush=True)
    if want("cfg5"):
        from oracle import exact
        for kappa in (1e2, 1e4, 1e6, 1e8):
            for eps in (1e-6, 1e-3, 1e-1):
                P = tlsgen.config(f"cfg5:k{kappa:g}:e{eps:g}", device="cuda", keep_factors=False)
                # the paper's constraint report D1-D8 (§3.1, oracle/exact.py) of this cell:
                # singular values from the construction, sigma_{n+1} from the SVD of the R factor of
                # [A, b], lambda_min(H) from the fp64 Gram (all on the GPU, not timed)
                Ab = torch.cat([P.A, P.b[:, None]], dim=1)
                Rab = torch.linalg.qr(Ab, mode="r")[1]
                sig_np1 = float(torch.linalg.svdvals(Rab)[-1])
                del Ab, Rab
                G = P.A.T @ P.A
                dd = 1.0 / torch.sqrt(torch.diagonal(G))
                lmin = float(torch.linalg.eigvalsh(G * dd[:, None] * dd[None, :])[0])
                del G
                s = P.s
                report = exact.constraint_report(P.m, P.n, s, sig_np1, float(np.linalg.norm(s)), lmin)
                for u_f in ("fp16", "bf16", "fp32", "fp64"):
                    rec = dense(P, u_f, 1)
                    u = UROUND[u_f]
                    # constr1: u_f * kappa(A) <~ 1 for the factorization
                    rec.update({"config": "cfg5", "kappa": kappa, "eps": eps,
                                "uf_times_kappa": u * kappa, "constr1_ok": u * kappa < 1.0,
                                "constraint_report": report,
                                "bounds_met": [k for k in ("D1", "D2", "D3", "D4", "D5", "D6", "D7", "D8")
                                               if u <= report[k]]})
                    sig = rec.get("sigma")
                    if sig is not None and math.isfinite(sig):
                        s_n = 1.0 / kappa
                        rec["sigma_over_sn"] = sig / s_n
                        rec["minimal"] = bool(sig < s_n)
                    res["runs"].append(rec)
                    print(json.dumps(rec), flush=True)
                del P
                torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
