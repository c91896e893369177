"""Where a cfg4w solve spends its device time, substitution vs explicit inverse (R24): the
library's per-category CUDA-event profile (tls_profile_*) of one whole tls_rqi_pcgtls on the
bench configuration, plus the unprofiled solve time (graph-captured loop).
python tools/prof_solve_split.py [cfg4w]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import tlsgen
from paper_2305_19028_b200 import tlsrqi as T
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4w"
torch.cuda.set_device(0)
P = tlsgen.config(name, device="cuda", keep_factors=False)
M = T.matrix(P.A)
ws = T.workspace(M)
rc, R, _ = T.tls_factor_precond(M, "fp16" if name != "cfg2w" else "bf16", ws=ws)
for pa in (1, 2):
    o = T.tls_rqi_opts_default(precond_apply=pa)
    T.tls_rqi_pcgtls(M, P.b, R, opts=o, ws=ws)
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc, x, sig, info = T.tls_rqi_pcgtls(M, P.b, R, opts=o, ws=ws)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    T.tls_profile_enable(True)
    rc, x, sig, info = T.tls_rqi_pcgtls(M, P.b, R, opts=o, ws=ws)
    torch.cuda.synchronize()
    prof = T.tls_profile_read()
    T.tls_profile_enable(False)
    parts = {k: (round(v["ms"], 3), v["count"]) for k, v in prof.items() if v["count"]}
    print(json.dumps({"workload": name, "precond_apply": pa, "solve_ms_unprofiled": round(min(ts), 3),
                      "profiled_sum_ms": round(sum(v["ms"] for v in prof.values()), 3),
                      "rqi": info["rqi_iters"], "boot": info["boot_iters"], "pcg": info["pcg_iters"],
                      "ms_count": parts}), flush=True)
