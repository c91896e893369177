"""GPU vs oracle on the full BASELINE cfg5 conditioning sweep (configs[4]: 65536 x 2048,
kappa in {1e2,1e4,1e6,1e8} x eps in {1e-6,1e-3,1e-1} x u_f in {fp16,bf16,fp32} plus the
u_f = fp64 control = 48 runs, VERDICT r01 missing #4).

Per run, on the same bytes (generated once per cell on the device, copied to the host):
  gpu       tls_factor_precond + tls_rqi_pcgtls through the C ABI
  oracle    the oracle's OWN pipeline (oracle.rqi.solve: its scaling, fp32-chunked Gram,
            LAPACK Cholesky, RQI-PCGTLS-MP)
  same_R    the oracle's RQI-PCGTLS-MP on the GPU's exported R~ (isolates the solve)
and the comparison: status, termination, RQI count, PCG counts (exact and within +-2),
bootstrap count, x (relative, 1e-9) and sigma (relative, 1e-12) when both are OK.

  python tools/cfg5_parity.py [--out gpurun_out/r02_cfg5_parity.jsonl] [--cells k1e2:e1e-6,...]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import tlsgen  # noqa: E402
from oracle import rqi  # noqa: E402
from paper_2305_19028_b200 import tlsrqi as T  # noqa: E402

STATUS = {v: k for k, v in vars(rqi).items() if k in ("OK", "CHOL_BREAKDOWN", "PCG_BREAKDOWN", "MAX_OUTER",
                                                       "NONFINITE", "RANGE", "NOT_MINIMAL", "STAGNATED")}


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def compare(g, o):
    """g: dict from the GPU, o: an oracle RqiResult (or a factor-only failure)."""
    out = {"status": g["status"] == o["status"], "termination": g.get("termination") == o.get("termination"),
           "rqi_iters": g.get("rqi_iters") == o.get("rqi_iters"),
           "pcg_exact": g.get("pcg_iters") == o.get("pcg_iters")}
    gp, op = g.get("pcg_iters") or [], o.get("pcg_iters") or []
    out["pcg_pm2"] = len(gp) == len(op) and all(abs(a[0] - b[0]) <= 2 and abs(a[1] - b[1]) <= 2 for a, b in zip(gp, op))
    out["boot_pm2"] = abs(g.get("boot_iters", 0) - o.get("boot_iters", 0)) <= 2
    if g["status"] == o["status"] == rqi.OK:
        out["x_rel"] = rel(g["x"], o["x"])
        out["sigma_rel"] = abs(g["sigma"] - o["sigma"]) / o["sigma"]
        out["x_ok"] = out["x_rel"] <= 1e-9
        out["sigma_ok"] = out["sigma_rel"] <= 1e-12
    return out


def orc_dict(pc, r):
    if pc is not None and pc.status != rqi.OK:
        return {"status": pc.status, "chol_pivot": pc.chol_pivot}
    return {"status": r.status, "termination": r.termination, "rqi_iters": r.rqi_iters, "boot_iters": r.boot_iters,
            "pcg_iters": [tuple(p) for p in r.pcg_iters], "x": r.x, "sigma": r.sigma}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/r02_cfg5_parity.jsonl")
    ap.add_argument("--cells", default="")
    ap.add_argument("--fmts", default="fp16,bf16,fp32,fp64")
    args = ap.parse_args()
    cells = [(k, e) for k in (1e2, 1e4, 1e6, 1e8) for e in (1e-6, 1e-3, 1e-1)]
    if args.cells:
        want = set(args.cells.split(","))
        cells = [c for c in cells if f"k{c[0]:g}:e{c[1]:g}" in want]
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    fo = open(args.out, "w")
    tally = {"runs": 0, "agree_status_term_K": 0, "agree_all": 0}
    for kappa, eps in cells:
        name = f"cfg5:k{kappa:g}:e{eps:g}"
        P = tlsgen.config(name, device="cuda", keep_factors=False)
        A = P.A.cpu().numpy()
        b = P.b.cpu().numpy()
        M = T.matrix(P.A)
        ws = T.workspace(M)
        for fmt in args.fmts.split(","):
            rec = {"cell": name, "u_f": fmt}
            rc, R, fi = T.tls_factor_precond(M, fmt, ws=ws)
            if R is None:
                g = {"status": rc, "chol_pivot": fi["chol_pivot"]}
            else:
                rc2, x, sig, info = T.tls_rqi_pcgtls(M, P.b, R, ws=ws)
                g = {"status": rc2, "termination": info["termination"], "rqi_iters": info["rqi_iters"],
                     "boot_iters": info["boot_iters"], "pcg_iters": [tuple(p) for p in info["pcg_iters"]],
                     "x": x.cpu().numpy(), "sigma": sig}
            t0 = time.time()
            pc, r = rqi.solve(A, b, fmt)
            rec["oracle_s"] = time.time() - t0
            o = orc_dict(pc, r)
            rec["gpu"] = {k: v for k, v in g.items() if k != "x"}
            rec["oracle"] = {k: v for k, v in o.items() if k != "x"}
            rec["vs_oracle"] = compare(g, o)
            if R is not None:
                Rt, d, nrm = T.tls_precond_export(R)
                rs = rqi.rqi_pcgtls_mp(A, b, rqi.Precond(Rt, d, fmt, nrm))
                rec["vs_oracle_same_R"] = compare(g, orc_dict(None, rs))
                iu = np.triu_indices(Rt.shape[0])
                if pc.status == rqi.OK:
                    rec["Rt_identical_frac"] = float(np.mean(Rt[iu] == pc.Rt[iu]))
            v = rec["vs_oracle"]
            tally["runs"] += 1
            core = v["status"] and (v["termination"] or g["status"] == rqi.CHOL_BREAKDOWN) and \
                (v["rqi_iters"] or g["status"] == rqi.CHOL_BREAKDOWN)
            tally["agree_status_term_K"] += int(core)
            tally["agree_all"] += int(core and v["pcg_pm2"] and v.get("x_ok", True) and v.get("sigma_ok", True))
            for key in ("gpu", "oracle"):
                rec[key]["status_name"] = STATUS.get(rec[key]["status"], str(rec[key]["status"]))
            print(json.dumps(rec, default=float), file=fo, flush=True)
            print(f"{name} {fmt}: gpu {rec['gpu']['status_name']} K={g.get('rqi_iters')} | oracle "
                  f"{rec['oracle']['status_name']} K={o.get('rqi_iters')} | {v} ({rec['oracle_s']:.1f}s)", flush=True)
        del P, M, ws
        torch.cuda.empty_cache()
    print(json.dumps({"summary": tally}), file=fo, flush=True)
    print("SUMMARY", tally, flush=True)


if __name__ == "__main__":
    main()
