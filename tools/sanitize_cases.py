"""Small invocations of every hand-synchronised kernel, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).  Run:

  compute-sanitizer --tool racecheck --target-processes all python tools/sanitize_cases.py [case ...]

Cases (all tiny so the instrumented run finishes in minutes):
  dense   cfg1-shaped fp16 factor (k_round_scaled, k_gram_tc, k_chol_dag, k_pack_R) + solve
          (k_pass ring, k_reduce_partials, trsv_ws clusters, k_pcg_*, k_rqi_*)
  chol    512 x 256 bf16 factor (k_chol_dag with several tile columns)
  winv    explicit-inverse solve (k_trtri, k_wpcg_step_coop, k_wgemv_grid)
  up32    u_p = fp32 solve (k_round32, k_pass32)
  csr     ragged CSR factor + solve (k_csr_*, k_csc_*)
  qr      Householder QR preconditioner, 1 leaf and TSQR (k_qr_*)
  f64     u_f = fp32 factor (k_gram_f64 DMMA)
Exit code 0 iff every case ran and returned its expected status.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import tlsgen  # noqa: E402
from paper_2305_19028_b200 import tlsrqi  # noqa: E402


def dense(P, u_f, **opts):
    A = torch.as_tensor(P.A, device="cuda")
    b = torch.as_tensor(P.b, device="cuda")
    M = tlsrqi.matrix(tlsrqi.dense_operand(A))
    rc, R, _ = tlsrqi.tls_factor_precond(M, u_f)
    assert rc == 0, rc
    o = tlsrqi.tls_rqi_opts_default(**opts) if opts else None
    rc, x, sig, info = tlsrqi.tls_rqi_pcgtls(M, b, R, opts=o)
    torch.cuda.synchronize()
    print(f"  {P.name} {u_f} {opts}: rc={rc} K={info['rqi_iters']} sigma={sig:.6e}", flush=True)
    return rc


def case_dense():
    assert dense(tlsgen.config("cfg1"), "fp16") == 0


def case_chol():
    P = tlsgen.dense_problem(512, 256, 1e2, 1e-3, 7, twin=True, name="d512x256")
    assert dense(P, "bf16") == 0


def case_winv():
    assert dense(tlsgen.config("cfg1"), "fp16", precond_apply=2) == 0


def case_up32():
    assert dense(tlsgen.config("cfg1"), "fp16", u_p="fp32") == 0


def case_csr():
    P = tlsgen.ragged_csr(600, 64, 50, 3)
    rp = torch.as_tensor(P.rowptr, device="cuda")
    ci = torch.as_tensor(P.colidx, device="cuda")
    va = torch.as_tensor(P.vals, device="cuda")
    b = torch.as_tensor(P.b, device="cuda")
    M = tlsrqi.matrix_csr(rp, ci, va, P.n)
    rc, R, _ = tlsrqi.tls_factor_precond(M, "fp16")
    assert rc == 0, rc
    rc, x, sig, info = tlsrqi.tls_rqi_pcgtls(M, b, R)
    torch.cuda.synchronize()
    print(f"  ragged csr: rc={rc} K={info['rqi_iters']}", flush=True)
    assert rc in (0, 7), rc


def case_qr():
    P = tlsgen.dense_problem(1024, 64, 1e2, 1e-3, 9, twin=True, name="qr")
    A = torch.as_tensor(P.A, device="cuda")
    M = tlsrqi.matrix(A)
    for leaves in ("1", "3"):
        os.environ["TLS_QR_LEAVES"] = leaves
        rc, R, _ = tlsrqi.tls_factor_precond_qr(M, "fp16")
        torch.cuda.synchronize()
        print(f"  qr leaves={leaves}: rc={rc}", flush=True)
        assert rc == 0, rc
    os.environ["TLS_QR_LEAVES"] = "1"


def case_f64():
    P = tlsgen.dense_problem(512, 128, 1e2, 1e-3, 11, twin=True, name="f64")
    assert dense(P, "fp32") == 0


CASES = {"dense": case_dense, "chol": case_chol, "winv": case_winv, "up32": case_up32,
         "csr": case_csr, "qr": case_qr, "f64": case_f64}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    torch.cuda.set_device(0)
    for nm in names:
        print(f"case {nm}", flush=True)
        CASES[nm]()
    print("ALL CASES OK", flush=True)
