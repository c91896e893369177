"""Time the preconditioner solves (tls_precond_apply: one CTA per RHS, warp-specialised
blocked TRSV) for several n and u_f with CUDA events; checks them against a dense
fp64 solve with torch on the GPU (triangular_solve), so it also catches a hang or a
wrong answer on the box before the parity suite runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2305_19028_b200 import tlsrqi

torch.cuda.set_device(0)
rng = np.random.default_rng(0)
for fmt, npdt in (("fp16", np.float16), ("bf16", None), ("fp32", np.float32), ("fp64", np.float64)):
    for n in (1024, 2048, 4096):
        R = np.triu(rng.standard_normal((n, n))) / n
        R[np.diag_indices(n)] = 1.0 + rng.random(n)
        if fmt == "bf16":
            R = torch.tensor(R).to(torch.bfloat16).double().numpy()
        else:
            R = R.astype(npdt).astype(np.float64)
        d = np.ldexp(1.0, rng.integers(-2, 3, n)).astype(np.float64)
        pc = tlsrqi.tls_precond_import(R, d, 1.0, fmt)
        Rt = torch.tensor(R, device="cuda") * torch.tensor(d, device="cuda")[None, :]  # P = R~ D
        for nrhs in (1, 2):
            for trans in (0, 1):
                Y0 = torch.randn((nrhs, n), dtype=torch.float64, device="cuda")
                Y = Y0.clone()
                tlsrqi.tls_precond_apply(pc, trans, Y)
                if trans == 0:
                    ref = torch.linalg.solve_triangular(Rt, Y0.T, upper=True).T
                else:
                    ref = torch.linalg.solve_triangular(Rt.T, Y0.T, upper=False).T
                err = float((Y - ref).norm() / ref.norm())
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                reps = 50
                e0.record()
                for _ in range(reps):
                    tlsrqi.tls_precond_apply(pc, trans, Y)
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) * 1e3 / reps
                print(f"{fmt:5s} n={n:5d} nrhs={nrhs} trans={trans}  {us:8.1f} us/apply  relerr {err:.2e}", flush=True)
