"""GPU parity of the CSR (cfg3) path through the C ABI against the CPU oracle.

Tolerances (tests/test_gpu_parity.py conventions):
  bit-exact        column scaling D; the fp16 CSR Gram (both sides: the exact sum of
                   the exact u_f products rounded once, reading R19); status, counts
  bound            bf16/fp32/fp64 CSR Gram (fp64 atomics): |G - G_oracle| <= 2 nnz_j u |A^|^T|A^|
  1e-12 relative   single passes (fp64, different summation order)
  1e-9 / 1e-12     x / sigma_{n+1} of a solve (north_star)
"""
import numpy as np
import pytest
import scipy.sparse
import torch

import tlsgen
from oracle import exact, rqi
from oracle.rounding import round_to

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def T():
    from paper_2305_19028_b200 import tlsrqi
    tlsrqi.lib()
    return tlsrqi


def _sp(P):
    return scipy.sparse.csr_matrix((P.vals, P.colidx, P.rowptr), shape=(P.m, P.n))


def _mat(T, P):
    rp = torch.as_tensor(P.rowptr, device="cuda")
    ci = torch.as_tensor(P.colidx.astype(np.int32), device="cuda")
    va = torch.as_tensor(P.vals, device="cuda")
    return T.matrix_csr(rp, ci, va, P.n)


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


PROBLEMS = {
    "cfg3_small": lambda: tlsgen.csr_problem(m=20000, n=400, per_row=10, seed=3),
    "ragged": lambda: tlsgen.ragged_csr(5000, 300, 70, seed=9),      # rows of 0..71 nnz (> 32: lane loops)
    "tall_narrow": lambda: tlsgen.csr_problem(m=3001, n=33, per_row=4, seed=2),
}


@pytest.mark.parametrize("name", sorted(PROBLEMS))
def test_csr_colstats_scaling_bitexact(T, name):
    P = PROBLEMS[name]()
    M = _mat(T, P)
    colmax, sumsq = T.tls_colstats(M)
    e = torch.frexp(colmax)[1]
    d_gpu = torch.ldexp(torch.ones_like(colmax), e - 1).cpu().numpy()
    d, normA2 = rqi.column_scaling(_sp(P))
    assert np.array_equal(d_gpu, d)
    assert float(sumsq) == pytest.approx(normA2, rel=1e-13)


@pytest.mark.parametrize("name", sorted(PROBLEMS))
@pytest.mark.parametrize("fmt", ["fp16", "bf16", "fp32", "fp64"])
def test_csr_gram(T, name, fmt):
    P = PROBLEMS[name]()
    A = _sp(P)
    d, _ = rqi.column_scaling(A)
    rc, G = T.tls_gram(_mat(T, P), fmt, torch.as_tensor(d, device="cuda"))
    assert rc == 0
    G = G.cpu().numpy()
    Go = rqi.gram_uf(A, d, fmt)
    if fmt == "fp16":
        assert np.array_equal(G, Go)            # exact sum rounded once on both sides (R19)
    else:
        Ah = A.copy()
        Ah.data = round_to(A.data / d[A.indices], fmt)
        absG = np.asarray((abs(Ah).T @ abs(Ah)).todense())
        cnt = np.asarray(((Ah != 0).astype(np.float64).T @ (Ah != 0).astype(np.float64)).todense())
        assert np.all(np.abs(G - Go) <= 2 * (cnt + 1) * 2.0 ** -53 * absG)
        assert np.array_equal(G, G.T)


@pytest.mark.parametrize("name", sorted(PROBLEMS))
def test_csr_passes(T, name):
    P = PROBLEMS[name]()
    A = _sp(P)
    M = _mat(T, P)
    rng = np.random.default_rng(1)
    q = rng.standard_normal((2, P.n))
    v, s = T.tls_pass(M, 0, torch.as_tensor(q, device="cuda"))
    v = v.cpu().numpy()
    s = s.cpu().numpy()
    for r in range(2):
        t = A @ q[r]
        assert _rel(v[r], A.T @ t) <= 1e-12
        assert s[r] == pytest.approx(t @ t, rel=1e-12)
    v1, s1 = T.tls_pass(M, 0, torch.as_tensor(q[:1], device="cuda"))
    t = A @ q[0]
    assert _rel(v1.cpu().numpy()[0], A.T @ t) <= 1e-12
    x = q[1]
    b = torch.as_tensor(P.b, device="cuda")
    vr, sr = T.tls_pass(M, 1, torch.as_tensor(x, device="cuda"), b)
    r = P.b - A @ x
    assert _rel(vr.cpu().numpy()[0], A.T @ r) <= 1e-12
    assert float(sr[0]) == pytest.approx(r @ r, rel=1e-12)
    assert float(sr[1]) == pytest.approx(P.b @ r, rel=1e-12)
    # deterministic: a second call gives identical bits
    v2, _ = T.tls_pass(M, 0, torch.as_tensor(q, device="cuda"))
    assert np.array_equal(v, v2.cpu().numpy())


def _check(info, x, sig, res, ex=None):
    assert info["status"] == res.status
    assert info["rqi_iters"] == res.rqi_iters
    assert info["boot_iters"] == res.boot_iters
    assert len(info["pcg_iters"]) == len(res.pcg_iters)
    for (a, b), (c, d) in zip(info["pcg_iters"], res.pcg_iters):
        assert abs(a - c) <= 2 and abs(b - d) <= 2
    if res.status == rqi.OK:
        assert _rel(x, res.x) <= 1e-9
        assert abs(sig - res.sigma) / res.sigma <= 1e-12
        if ex is not None:
            assert _rel(x, ex.x) <= 1e-9
            assert abs(sig - ex.sigma) / ex.sigma <= 1e-11


@pytest.mark.parametrize("fmt", ["fp16", "bf16", "fp32"])
def test_csr_solve_end_to_end(T, fmt):
    P = PROBLEMS["cfg3_small"]()
    A = _sp(P)
    M = _mat(T, P)
    rc, R, _ = T.tls_factor_precond(M, fmt)
    assert rc == 0
    rc, x, sig, info = T.tls_rqi_pcgtls(M, torch.as_tensor(P.b, device="cuda"), R)
    pc, res = rqi.solve(A, P.b, fmt)
    if fmt == "fp16":
        # same Gram bits; R~ from two Cholesky implementations agrees to within one ulp
        Rt, d, _ = T.tls_precond_export(R)
        ulp = np.spacing(np.abs(pc.Rt).astype(np.float16)).astype(np.float64)
        assert np.all(np.abs(Rt - pc.Rt) <= ulp)
    ex = exact.tls_svd(P.to_dense(), P.b)
    _check(info, x.cpu().numpy(), sig, res, ex)


def test_csr_solve_imported_R_ragged(T):
    P = PROBLEMS["ragged"]()
    A = _sp(P)
    pc, res = rqi.solve(A, P.b, "fp16")
    R = T.tls_precond_import(pc.Rt, pc.d, pc.normA2, "fp16")
    rc, x, sig, info = T.tls_rqi_pcgtls(_mat(T, P), torch.as_tensor(P.b, device="cuda"), R)
    _check(info, x.cpu().numpy(), sig, res, exact.tls_svd(P.to_dense(), P.b))


def test_cfg3_full_size(T):
    """BASELINE configs[2] at full size (200000 x 2000, 2.2M nnz, u_f fp16):
    GPU factor + solve vs the oracle's pipeline on the same CSR bytes."""
    P = tlsgen.config("cfg3")
    A = _sp(P)
    M = _mat(T, P)
    rc, R, _ = T.tls_factor_precond(M, "fp16")
    assert rc == 0
    rc, x, sig, info = T.tls_rqi_pcgtls(M, torch.as_tensor(P.b, device="cuda"), R)
    pc, res = rqi.solve(A, P.b, "fp16")
    _check(info, x.cpu().numpy(), sig, res)
    assert res.status == rqi.OK
    # minimality certificate on the oracle side: sigma below the smallest singular value of A
    assert res.sigma < np.sqrt(np.linalg.eigvalsh(np.asarray((A.T @ A).todense()))[0])
