"""ctypes binding of libtlsrqi.so (include/tlsrqi.h) — argument marshalling only.

Every function here has the name of the C entry point it calls and does no
numerical work: all steps of RQI-PCGTLS-MP run in the CUDA kernels of the
library.  PyTorch is used for device memory and streams.  If the shared
library is missing the import of the functions raises (no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtlsrqi.so")

TLS_FP16, TLS_BF16, TLS_FP32, TLS_FP64 = 0, 1, 2, 3
PREC = {"fp16": TLS_FP16, "bf16": TLS_BF16, "fp32": TLS_FP32, "fp64": TLS_FP64}
TLS_DENSE_ROWMAJOR, TLS_CSR = 0, 1
STATUS = {0: "OK", 1: "CHOL_BREAKDOWN", 2: "PCG_BREAKDOWN", 3: "MAX_OUTER", 4: "NONFINITE",
          5: "RANGE", 6: "NOT_MINIMAL", 7: "STAGNATED", -1: "ERR_ARG", -2: "ERR_CUDA",
          -3: "ERR_NCCL", -4: "ERR_WORKSPACE", -5: "ERR_UNSUPPORTED"}
TERM = {0: "NONE", 1: "CONVERGED_TOL", 2: "PSI_INCREASE_CONVERGED", 3: "STAGNATED",
        4: "MAX_OUTER", 5: "BREAKDOWN", 6: "NONFINITE"}


class tls_matrix_t(C.Structure):
    _fields_ = [("layout", C.c_int32), ("reserved", C.c_int32), ("m_local", C.c_int64),
                ("n", C.c_int64), ("m_global", C.c_int64), ("row_offset", C.c_int64),
                ("ld", C.c_int64), ("vals", C.c_void_p), ("rowptr", C.c_void_p),
                ("colidx", C.c_void_p), ("nnz_local", C.c_int64)]


class tls_rqi_opts_t(C.Structure):
    _fields_ = [("budget_rule", C.c_int32), ("stop_rule", C.c_int32), ("max_outer", C.c_int32),
                ("polish", C.c_int32), ("tol_inner", C.c_double), ("boot", C.c_int32),
                ("boot_max", C.c_int32), ("boot_tol", C.c_double), ("op_variant", C.c_int32),
                ("breakdown_rule", C.c_int32), ("gram_chunk", C.c_int32), ("u_p", C.c_int32),
                ("precond_apply", C.c_int32), ("certify", C.c_int32), ("minimal_check", C.c_int32),
                ("reserved", C.c_int32)]


class tls_info_t(C.Structure):
    _fields_ = [("status", C.c_int32), ("termination", C.c_int32), ("rqi_iters", C.c_int32),
                ("boot_iters", C.c_int32), ("pcg_iters", C.POINTER(C.c_int32)),
                ("sigma2_trace", C.POINTER(C.c_double)), ("psi_trace", C.POINTER(C.c_double)),
                ("breakdown_k", C.c_int32), ("breakdown_rhs", C.c_int32),
                ("breakdown_j", C.c_int32), ("chol_pivot", C.c_int32), ("sigma2", C.c_double),
                ("passes", C.c_int64), ("launches", C.c_int32), ("pcg_steps", C.c_int32),
                ("sigma_certified", C.c_double), ("delta_min_trace", C.POINTER(C.c_double))]


_lib = None


def lib() -> C.CDLL:
    """Load libtlsrqi.so (raises if it has not been built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2305_19028_b200.build`")
    L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    P, VP, I32, I64, D, SZ = C.POINTER, C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_size_t
    M = P(tls_matrix_t)
    sig = {
        "tls_abi_version": (C.c_int, []),
        "tls_rqi_opts_default": (None, [P(tls_rqi_opts_t)]),
        "tls_status_string": (C.c_char_p, [C.c_int]),
        "tls_last_error": (C.c_char_p, []),
        "tls_comm_get_unique_id": (C.c_int, [VP]),
        "tls_comm_init": (C.c_int, [C.c_int, C.c_int, VP, C.c_int, P(VP)]),
        "tls_comm_destroy": (C.c_int, [VP]),
        "tls_comm_init_shm": (C.c_int, [C.c_int, C.c_int, C.c_char_p, SZ, C.c_int, P(VP)]),
        "tls_comm_nranks": (C.c_int, [VP]),
        "tls_comm_rank": (C.c_int, [VP]),
        "tls_comm_peer_prepare": (C.c_int, [VP, I64, VP]),
        "tls_comm_peer_connect": (C.c_int, [VP, VP]),
        "tls_peer_exchange_emulate": (C.c_int, [C.c_int, VP, C.c_int, C.c_int, C.c_int, VP, VP]),
        "tls_workspace_size": (SZ, [M, I32]),
        "tls_factor_precond": (C.c_int, [M, I32, P(tls_rqi_opts_t), VP, VP, VP, SZ, P(VP), P(tls_info_t)]),
        "tls_qr_workspace_size": (SZ, [M, I32, I32]),
        "tls_factor_precond_qr": (C.c_int, [M, I32, VP, VP, VP, SZ, P(VP), P(tls_info_t)]),
        "tls_qr_blocked_workspace_size": (SZ, [M, I32]),
        "tls_factor_precond_qr_blocked": (C.c_int, [M, I32, VP, VP, SZ, P(VP), P(tls_info_t)]),
        "tls_precond_import": (C.c_int, [I64, I32, VP, VP, D, VP, P(VP)]),
        "tls_precond_export": (C.c_int, [VP, VP, VP, P(D)]),
        "tls_precond_destroy": (None, [VP]),
        "tls_precond_prepare": (C.c_int, [M, VP, I32, VP, VP, SZ]),
        "tls_rqi_pcgtls": (C.c_int, [M, VP, VP, I32, I32, D, P(tls_rqi_opts_t), VP, VP, VP, SZ, VP,
                                     P(D), P(tls_info_t)]),
        "tls_solve_host_bytes": (SZ, [I64, I64, I64, I32]),
        "tls_solve_host": (C.c_int, [VP, VP, I64, I64, I64, I64, I64, I32, D, P(tls_rqi_opts_t), VP,
                                     VP, VP, SZ, VP, P(D), P(tls_info_t)]),
        "tls_colstats": (C.c_int, [M, VP, VP, VP, VP, SZ]),
        "tls_gram": (C.c_int, [M, I32, VP, I32, VP, VP, VP, SZ]),
        "tls_pass": (C.c_int, [M, I32, I32, VP, VP, VP, VP, VP, VP, SZ]),
        "tls_pass_fp32": (C.c_int, [M, VP, VP, VP, VP, VP, VP, SZ]),
        "tls_precond_apply": (C.c_int, [VP, I32, I32, VP, VP]),
        "tls_round": (C.c_int, [VP, VP, I64, I32, VP]),
        "tls_profile_enable": (C.c_int, [C.c_int]),
        "tls_profile_read": (C.c_int, [P(D), P(I64), C.c_int]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


EXPORTED = ["tls_abi_version", "tls_rqi_opts_default", "tls_status_string", "tls_last_error",
            "tls_comm_get_unique_id", "tls_comm_init", "tls_comm_init_shm", "tls_comm_nranks", "tls_comm_rank",
            "tls_comm_peer_prepare", "tls_comm_peer_connect", "tls_peer_exchange_emulate",
            "tls_comm_destroy", "tls_workspace_size",
            "tls_factor_precond", "tls_qr_workspace_size", "tls_factor_precond_qr", "tls_qr_blocked_workspace_size",
            "tls_factor_precond_qr_blocked", "tls_precond_import", "tls_precond_export", "tls_precond_destroy",
            "tls_precond_prepare",
            "tls_rqi_pcgtls", "tls_solve_host_bytes", "tls_solve_host", "tls_colstats", "tls_gram",
            "tls_pass", "tls_pass_fp32", "tls_precond_apply", "tls_round", "tls_profile_enable", "tls_profile_read"]

PROF_CATS = ["pass_op2", "pass_op1", "pass_resid", "colstats", "gram", "chol", "pcg_step",
             "pcg_init", "reduce", "pass_op2_fp32"]


class TlsError(RuntimeError):
    def __init__(self, rc: int, where: str):
        msg = lib().tls_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS.get(rc, rc)} ({msg})")
        self.rc = rc


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream) -> C.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _check(rc: int, where: str) -> int:
    if rc < 0:
        raise TlsError(rc, where)
    return rc


def tls_status_string(rc: int) -> str:
    return lib().tls_status_string(rc).decode()


def tls_rqi_opts_default(**over) -> tls_rqi_opts_t:
    o = tls_rqi_opts_t()
    lib().tls_rqi_opts_default(C.byref(o))
    for k, v in over.items():
        if k == "u_p" and isinstance(v, str):      # "fp64" / "fp32" (R23)
            v = PREC[v]
        setattr(o, k, v)
    return o


def matrix(A: torch.Tensor, m_global: Optional[int] = None, row_offset: int = 0, n: Optional[int] = None):
    """tls_matrix_t for a row-major fp64 CUDA tensor (m_local x ld, ld even)."""
    assert A.is_cuda and A.dtype == torch.float64 and A.dim() == 2 and A.stride(1) == 1
    m, ld = A.shape[0], A.stride(0)
    nn = A.shape[1] if n is None else n
    M = tls_matrix_t()
    M.layout = TLS_DENSE_ROWMAJOR
    M.m_local, M.n, M.ld = m, nn, ld
    M.m_global = m if m_global is None else m_global
    M.row_offset = row_offset
    M.vals = A.data_ptr()
    M._keep = A            # the descriptor keeps its device buffer alive
    return M


def matrix_csr(rowptr: torch.Tensor, colidx: torch.Tensor, vals: torch.Tensor, n: int,
               m_global: Optional[int] = None, row_offset: int = 0):
    """tls_matrix_t for a CSR row block on the device: rowptr int64 (m_local + 1,
    rowptr[0] = 0), colidx int32 (ascending within a row), vals fp64."""
    assert rowptr.is_cuda and rowptr.dtype == torch.int64 and rowptr.dim() == 1
    assert colidx.is_cuda and colidx.dtype == torch.int32 and vals.is_cuda and vals.dtype == torch.float64
    assert colidx.numel() == vals.numel()
    m = rowptr.numel() - 1
    M = tls_matrix_t()
    M.layout = TLS_CSR
    M.m_local, M.n, M.ld = m, n, 0
    M.m_global = m if m_global is None else m_global
    M.row_offset = row_offset
    M.rowptr = rowptr.data_ptr()
    M.colidx = colidx.data_ptr() if colidx.numel() else None
    M.vals = vals.data_ptr() if vals.numel() else None
    M.nnz_local = vals.numel()
    M._keep = (rowptr, colidx, vals)
    return M


def dense_operand(A: torch.Tensor) -> torch.Tensor:
    """Row-major fp64 copy with an even leading dimension (pads one zero column if n is odd)."""
    A = A.to(torch.float64)
    m, n = A.shape
    if n % 2 == 0 and A.is_contiguous():
        return A
    ld = n + (n % 2)
    out = torch.zeros((m, ld), dtype=torch.float64, device=A.device)
    out[:, :n] = A
    return out[:, :n] if ld == n else out.as_strided((m, n), (ld, 1))


def tls_workspace_size(M: tls_matrix_t, max_outer: int = 50) -> int:
    return int(lib().tls_workspace_size(C.byref(M), max_outer))


def workspace(M: tls_matrix_t, device=None) -> torch.Tensor:
    nbytes = tls_workspace_size(M)
    if nbytes == 0:
        raise TlsError(-1, "tls_workspace_size")
    return torch.empty(nbytes, dtype=torch.uint8, device=device or "cuda")


def _info(max_outer: int):
    info = tls_info_t()
    pcg = (C.c_int32 * (2 * max_outer + 2))()
    s2 = (C.c_double * (max_outer + 2))()
    ps = (C.c_double * (max_outer + 2))()
    dm = (C.c_double * (2 * max_outer + 2))()
    info.pcg_iters = C.cast(pcg, C.POINTER(C.c_int32))
    info.sigma2_trace = C.cast(s2, C.POINTER(C.c_double))
    info.psi_trace = C.cast(ps, C.POINTER(C.c_double))
    info.delta_min_trace = C.cast(dm, C.POINTER(C.c_double))
    return info, (pcg, s2, ps, dm)


def _info_dict(info: tls_info_t, bufs) -> dict:
    pcg, s2, ps, dm = bufs
    k = max(int(info.rqi_iters), 0)
    npcg = max(int(info.pcg_steps), 0)
    return {
        "status": int(info.status), "status_name": STATUS.get(int(info.status), "?"),
        "termination": int(info.termination), "termination_name": TERM.get(int(info.termination), "?"),
        "rqi_iters": k, "boot_iters": int(info.boot_iters),
        "pcg_iters": [(pcg[2 * i], pcg[2 * i + 1]) for i in range(npcg)],
        "sigma2_trace": [s2[i] for i in range(k)], "psi_trace": [ps[i] for i in range(k)],
        "breakdown_k": int(info.breakdown_k), "breakdown_rhs": int(info.breakdown_rhs),
        "breakdown_j": int(info.breakdown_j), "chol_pivot": int(info.chol_pivot),
        "sigma2": float(info.sigma2), "passes": int(info.passes), "launches": int(info.launches),
        "sigma_certified": float(info.sigma_certified),
        "delta_min_trace": [(dm[2 * i], dm[2 * i + 1]) for i in range(npcg)],
    }


class Precond:
    """Owning wrapper of a tls_precond_t handle."""

    def __init__(self, handle: int, n: int, u_f: int):
        self.handle, self.n, self.u_f = handle, n, u_f

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.tls_precond_destroy(C.c_void_p(self.handle))
            self.handle = None


def tls_factor_precond(M: tls_matrix_t, u_f, opts: Optional[tls_rqi_opts_t] = None, comm=None,
                       stream=None, ws: Optional[torch.Tensor] = None):
    """Returns (status, Precond or None, info dict)."""
    uf = PREC[u_f] if isinstance(u_f, str) else int(u_f)
    if ws is None:
        ws = workspace(M)
    R = C.c_void_p()
    info, bufs = _info(opts.max_outer if opts else 50)
    rc = lib().tls_factor_precond(C.byref(M), uf, C.byref(opts) if opts else None,
                                  C.c_void_p(comm) if comm else None, _stream(stream),
                                  _ptr(ws), ws.numel(), C.byref(R), C.byref(info))
    _check(rc, "tls_factor_precond")
    d = _info_dict(info, bufs)
    return rc, (Precond(R.value, int(M.n), uf) if R.value else None), d


def tls_factor_precond_qr(M: tls_matrix_t, u_f, comm=None, stream=None, ws: Optional[torch.Tensor] = None,
                          nranks: Optional[int] = None):
    """Householder-QR preconditioner in u_f (NEXT-2, R25; TSQR over ranks / TLS_QR_LEAVES, R26).
    nranks: sizes the TSQR stack in the workspace when ws is None; default: the size of
    `comm` (tls_comm_nranks), 1 without one.
    Returns (status, Precond or None, info dict)."""
    uf = PREC[u_f] if isinstance(u_f, str) else int(u_f)
    if nranks is None:
        nranks = int(lib().tls_comm_nranks(C.c_void_p(comm) if comm else None))
    if ws is None:
        nbytes = int(lib().tls_qr_workspace_size(C.byref(M), uf, nranks))
        if nbytes == 0:
            raise TlsError(-1, "tls_qr_workspace_size")
        ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    R = C.c_void_p()
    info, bufs = _info(50)
    rc = lib().tls_factor_precond_qr(C.byref(M), uf, C.c_void_p(comm) if comm else None, _stream(stream),
                                     _ptr(ws), ws.numel(), C.byref(R), C.byref(info))
    _check(rc, "tls_factor_precond_qr")
    return rc, (Precond(R.value, int(M.n), uf) if R.value else None), _info_dict(info, bufs)


def tls_factor_precond_qr_blocked(M: tls_matrix_t, u_f, stream=None, ws: Optional[torch.Tensor] = None):
    """Blocked Householder QR in u_f with tensor-core WY trailing updates (R29, NEXT-2).
    Returns (status, Precond or None, info dict)."""
    uf = PREC[u_f] if isinstance(u_f, str) else int(u_f)
    if ws is None:
        nbytes = int(lib().tls_qr_blocked_workspace_size(C.byref(M), uf))
        if nbytes == 0:
            raise TlsError(-1, "tls_qr_blocked_workspace_size")
        ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    R = C.c_void_p()
    info, bufs = _info(50)
    rc = lib().tls_factor_precond_qr_blocked(C.byref(M), uf, _stream(stream), _ptr(ws), ws.numel(), C.byref(R),
                                             C.byref(info))
    _check(rc, "tls_factor_precond_qr_blocked")
    return rc, (Precond(R.value, int(M.n), uf) if R.value else None), _info_dict(info, bufs)


def tls_precond_import(Rt, d, normA2: float, u_f, stream=None) -> Precond:
    import numpy as np
    Rt = np.ascontiguousarray(Rt, dtype=np.float64)
    d = np.ascontiguousarray(d, dtype=np.float64)
    uf = PREC[u_f] if isinstance(u_f, str) else int(u_f)
    R = C.c_void_p()
    rc = lib().tls_precond_import(Rt.shape[0], uf, Rt.ctypes.data_as(C.c_void_p),
                                  d.ctypes.data_as(C.c_void_p), float(normA2), _stream(stream), C.byref(R))
    if rc != 0:
        raise TlsError(rc, "tls_precond_import")
    return Precond(R.value, Rt.shape[0], uf)


def tls_precond_prepare(M: tls_matrix_t, R: Precond, what: int = 3, stream=None, ws: Optional[torch.Tensor] = None):
    """Make R's solve-time buffers now (1: explicit inverse W, 2: fp32 copy of A, 3: both), so that
    tls_rqi_pcgtls allocates nothing (tlsrqi.h)."""
    if ws is None and what & 2:
        ws = workspace(M)
    _check(lib().tls_precond_prepare(C.byref(M), C.c_void_p(R.handle), int(what), _stream(stream), _ptr(ws),
                                     0 if ws is None else ws.numel()), "tls_precond_prepare")


def tls_precond_export(R: Precond):
    import numpy as np
    Rt = np.zeros((R.n, R.n))
    d = np.zeros(R.n)
    nrm = C.c_double()
    _check(lib().tls_precond_export(C.c_void_p(R.handle), Rt.ctypes.data_as(C.c_void_p),
                                    d.ctypes.data_as(C.c_void_p), C.byref(nrm)), "tls_precond_export")
    return Rt, d, nrm.value


def tls_rqi_pcgtls(M: tls_matrix_t, b: torch.Tensor, R: Precond, tol: float = 1e-14,
                   opts: Optional[tls_rqi_opts_t] = None, comm=None, stream=None,
                   ws: Optional[torch.Tensor] = None, x_out: Optional[torch.Tensor] = None,
                   u: int = TLS_FP64, u_r: int = TLS_FP64):
    """Returns (status, x (device tensor), sigma, info dict)."""
    if ws is None:
        ws = workspace(M)
    if x_out is None:
        x_out = torch.empty(int(M.n), dtype=torch.float64, device=b.device)
    sigma = C.c_double()
    info, bufs = _info(opts.max_outer if opts else 50)
    rc = lib().tls_rqi_pcgtls(C.byref(M), _ptr(b), C.c_void_p(R.handle), u, u_r, tol,
                              C.byref(opts) if opts else None, C.c_void_p(comm) if comm else None,
                              _stream(stream), _ptr(ws), ws.numel(), _ptr(x_out), C.byref(sigma),
                              C.byref(info))
    _check(rc, "tls_rqi_pcgtls")
    return rc, x_out, sigma.value, _info_dict(info, bufs)


def tls_solve_host_bytes(m: int, n: int, ld: int, max_outer: int = 50) -> int:
    return int(lib().tls_solve_host_bytes(m, n, ld, max_outer))


def tls_solve_host(A_host: torch.Tensor, b_host: torch.Tensor, u_f, tol: float = 1e-14,
                   opts: Optional[tls_rqi_opts_t] = None, dev_buf: Optional[torch.Tensor] = None,
                   stream=None, x_host: Optional[torch.Tensor] = None, comm=None,
                   m_global: Optional[int] = None, row_offset: int = 0):
    """End to end from host (ideally pinned) buffers.  Returns (status, x_host, sigma, info)."""
    assert A_host.device.type == "cpu" and A_host.dtype == torch.float64 and A_host.stride(1) == 1
    m, n = A_host.shape
    ld = A_host.stride(0)
    if dev_buf is None:
        dev_buf = torch.empty(tls_solve_host_bytes(m, n, ld), dtype=torch.uint8, device="cuda")
    if x_host is None:
        x_host = torch.empty(n, dtype=torch.float64).pin_memory()
    uf = PREC[u_f] if isinstance(u_f, str) else int(u_f)
    sigma = C.c_double()
    info, bufs = _info(opts.max_outer if opts else 50)
    rc = lib().tls_solve_host(_ptr(A_host), _ptr(b_host), m, n, ld, m if m_global is None else m_global,
                              row_offset, uf, tol, C.byref(opts) if opts else None,
                              C.c_void_p(comm) if comm else None, _stream(stream), _ptr(dev_buf),
                              dev_buf.numel(), _ptr(x_host), C.byref(sigma), C.byref(info))
    _check(rc, "tls_solve_host")
    return rc, x_host, sigma.value, _info_dict(info, bufs)


def tls_colstats(M: tls_matrix_t, stream=None, ws=None):
    if ws is None:
        ws = workspace(M)
    colmax = torch.empty(int(M.n), dtype=torch.float64, device="cuda")
    sumsq = torch.empty(1, dtype=torch.float64, device="cuda")
    _check(lib().tls_colstats(C.byref(M), _ptr(colmax), _ptr(sumsq), _stream(stream), _ptr(ws),
                              ws.numel()), "tls_colstats")
    return colmax, sumsq


def tls_gram(M: tls_matrix_t, u_f, d: torch.Tensor, K_t: int = 64, stream=None, ws=None):
    if ws is None:
        ws = workspace(M)
    n = int(M.n)
    G = torch.empty((n, n), dtype=torch.float64, device="cuda")
    uf = PREC[u_f] if isinstance(u_f, str) else int(u_f)
    rc = _check(lib().tls_gram(C.byref(M), uf, _ptr(d), K_t, _ptr(G), _stream(stream), _ptr(ws),
                               ws.numel()), "tls_gram")
    return rc, G


def tls_pass(M: tls_matrix_t, mode: int, q: torch.Tensor, b: Optional[torch.Tensor] = None,
             stream=None, ws=None):
    """mode 0: (v = A^T A q_r, s_r = ||A q_r||^2); mode 1: (v = A^T(b - A q), [r^T r, b^T r])."""
    if ws is None:
        ws = workspace(M)
    nrhs = 1 if q.dim() == 1 else q.shape[0]
    v = torch.empty((nrhs, int(M.n)), dtype=torch.float64, device="cuda")
    s = torch.empty(2, dtype=torch.float64, device="cuda")
    _check(lib().tls_pass(C.byref(M), mode, nrhs, _ptr(q.contiguous()), _ptr(b), _ptr(v), _ptr(s),
                          _stream(stream), _ptr(ws), ws.numel()), "tls_pass")
    return v, s


def tls_pass_fp32(M: tls_matrix_t, R: "Precond", q: torch.Tensor, stream=None, ws=None):
    """u_p = fp32 operator pass (R23) on R's fp32 copy of A: q (2 x n) -> (v, s)."""
    if ws is None:
        ws = workspace(M)
    v = torch.empty((2, int(M.n)), dtype=torch.float64, device="cuda")
    s = torch.empty(2, dtype=torch.float64, device="cuda")
    _check(lib().tls_pass_fp32(C.byref(M), C.c_void_p(R.handle), _ptr(q.contiguous()), _ptr(v), _ptr(s),
                               _stream(stream), _ptr(ws), ws.numel()), "tls_pass_fp32")
    return v, s


def tls_precond_apply(R: Precond, trans: int, Y: torch.Tensor, stream=None) -> torch.Tensor:
    """In place: Y (nrhs x n) <- P^{-1} Y (trans 0) or P^{-T} Y (trans 1); trans | 2 applies
    them through the explicit inverse W = R~^{-1} (R24)."""
    nrhs = 1 if Y.dim() == 1 else Y.shape[0]
    assert Y.is_contiguous()
    _check(lib().tls_precond_apply(C.c_void_p(R.handle), trans, nrhs, _ptr(Y), _stream(stream)),
           "tls_precond_apply")
    return Y


def tls_round(x: torch.Tensor, prec, stream=None) -> torch.Tensor:
    y = torch.empty_like(x)
    p = PREC[prec] if isinstance(prec, str) else int(prec)
    _check(lib().tls_round(_ptr(x), _ptr(y), x.numel(), p, _stream(stream)), "tls_round")
    return y


def tls_comm_get_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(lib().tls_comm_get_unique_id(buf), "tls_comm_get_unique_id")
    return bytes(buf)


def tls_comm_init(nranks: int, rank: int, uid: bytes, device: int) -> int:
    h = C.c_void_p()
    buf = (C.c_char * 128).from_buffer_copy(uid)
    _check(lib().tls_comm_init(nranks, rank, buf, device, C.byref(h)), "tls_comm_init")
    return h.value


def tls_comm_init_shm(nranks: int, rank: int, name: str, device: int, slot_bytes: int = 1 << 22) -> int:
    """Host-staged communicator for ranks sharing one GPU (tlsrqi.h tls_comm_init_shm)."""
    h = C.c_void_p()
    _check(lib().tls_comm_init_shm(nranks, rank, name.encode(), slot_bytes, device, C.byref(h)), "tls_comm_init_shm")
    return h.value


def tls_comm_peer_prepare(comm: int, wcap: int) -> bytes:
    """This rank's 128-byte CUDA-IPC record of its peer-exchange buffers (tlsrqi.h)."""
    buf = (C.c_char * 128)()
    _check(lib().tls_comm_peer_prepare(C.c_void_p(comm), int(wcap), buf), "tls_comm_peer_prepare")
    return bytes(buf)


def tls_comm_peer_connect(comm: int, records) -> None:
    """Map every rank's buffers; `records` = the ranks' 128-byte records in rank order."""
    blob = b"".join(records)
    if len(blob) != 128 * len(records):
        raise ValueError("peer records must be 128 bytes each")
    _check(lib().tls_comm_peer_connect(C.c_void_p(comm), C.create_string_buffer(blob, len(blob))),
           "tls_comm_peer_connect")


def comm_attach_peer(comm: int, wcap: int, group=None) -> None:
    """NEXT-3 peer exchange on a communicator whose ranks are processes on DIFFERENT GPUs:
    prepare, all-gather the ranks' records with torch.distributed (rank order), connect."""
    import torch.distributed as dist
    rec = tls_comm_peer_prepare(comm, wcap)
    recs = [None] * dist.get_world_size(group)
    dist.all_gather_object(recs, rec, group=group)
    tls_comm_peer_connect(comm, recs)


def tls_peer_exchange_emulate(partials: torch.Tensor, reps: int = 1, stream=None) -> torch.Tensor:
    """Test hook: the exchange kernel for P emulated ranks in one cooperative launch on this GPU.
    partials: [P, G, W] fp64 CUDA tensor; returns [P, W] (every rank's pass sums)."""
    assert partials.is_cuda and partials.dtype == torch.float64 and partials.dim() == 3 and partials.is_contiguous()
    P, G, W = partials.shape
    out = torch.empty((P, W), dtype=torch.float64, device=partials.device)
    _check(lib().tls_peer_exchange_emulate(P, _ptr(partials), G, W, reps, _ptr(out), _stream(stream)),
           "tls_peer_exchange_emulate")
    return out


def tls_comm_nranks(comm) -> int:
    return int(lib().tls_comm_nranks(C.c_void_p(comm) if comm else None))


def tls_comm_destroy(comm: int) -> None:
    lib().tls_comm_destroy(C.c_void_p(comm))


def tls_profile_enable(on: bool = True) -> None:
    lib().tls_profile_enable(1 if on else 0)


def tls_profile_read() -> dict:
    n = len(PROF_CATS)
    ms = (C.c_double * n)()
    cnt = (C.c_int64 * n)()
    lib().tls_profile_read(ms, cnt, n)
    return {k: {"ms": ms[i], "count": int(cnt[i])} for i, k in enumerate(PROF_CATS)}
