"""The paper's E5 comparison (on Van Huffel's problem the QR preconditioner
needs several times more RQI steps than the Cholesky one) over all five §4 problems, through
the GPU path: status, RQI steps and total PCG iterations with each preconditioner, u_f in
{fp16, bf16} and the fp64 control (the paper's RQI-PCGTLS).  Writes a table to stdout."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import tlsgen
from paper_2305_19028_b200 import tlsrqi as T

print(f"{'problem':10s} {'u_f':5s} | {'chol: status':>14s} {'RQI':>4s} {'PCG':>5s} | {'qr: status':>14s} {'RQI':>4s} {'PCG':>5s}")
for name in tlsgen.PAPER_PROBLEMS:
    P = tlsgen.paper_problem(name)
    A = torch.as_tensor(np.ascontiguousarray(P.A), device="cuda")
    M = T.matrix(T.dense_operand(A), n=P.n)
    b = torch.as_tensor(P.b, device="cuda")
    for fmt in ("fp16", "bf16", "fp64"):     # fp64: RQI-PCGTLS, the paper's fixed-precision reference
        cells = []
        for fac in (T.tls_factor_precond, T.tls_factor_precond_qr):
            rc, R, fi = fac(M, fmt)
            if rc != 0:
                cells.append((f"factor {T.STATUS.get(rc, rc)}", "-", "-"))
                continue
            rc, x, sig, info = T.tls_rqi_pcgtls(M, b, R)
            pcg = sum(p[0] for p in info["pcg_iters"])
            cells.append((info["status_name"], info["rqi_iters"], pcg))
        print(f"{name:10s} {fmt:5s} | {cells[0][0]:>14s} {cells[0][1]!s:>4s} {cells[0][2]!s:>5s} | "
              f"{cells[1][0]:>14s} {cells[1][1]!s:>4s} {cells[1][2]!s:>5s}", flush=True)
