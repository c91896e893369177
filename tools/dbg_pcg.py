"""Debug driver: step-by-step solves with a watchdog (prints progress; used on the box)."""
import os, sys, time, faulthandler
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(int(os.environ.get("DBG_T", 60)), exit=True)
import numpy as np, torch
import tlsgen
from oracle import rqi
from paper_2305_19028_b200 import tlsrqi as T
for name, fmt in [("cfg1", "fp16"), ("cfg2w", "fp16"), ("cfg2w", "bf16")]:
    P = tlsgen.config(name)
    pc = rqi.factor_precond(P.A, fmt)
    R = T.tls_precond_import(pc.Rt, pc.d, pc.normA2, fmt)
    M = T.matrix(torch.as_tensor(P.A, device="cuda"))
    b = torch.as_tensor(P.b, device="cuda")
    for boot_max in (1, 2, 8, 200):
        o = T.tls_rqi_opts_default(boot_max=boot_max, max_outer=3)
        t = time.time()
        rc, x, sig, info = T.tls_rqi_pcgtls(M, b, R, opts=o)
        torch.cuda.synchronize()
        print(name, fmt, "boot_max", boot_max, "rc", rc, info["boot_iters"], info["rqi_iters"], info["pcg_iters"], f"{time.time()-t:.3f}s", flush=True)
