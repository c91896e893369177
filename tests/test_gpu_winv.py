"""GPU parity of the explicit-inverse preconditioner application (reading R24,
tls_rqi_opts_t.precond_apply = 2): k_trtri's W = R~^{-1} and the cluster GEMVs that
replace the substitutions, against oracle.rqi.with_inverse / RqiOptions(precond_apply=2)."""
import numpy as np
import pytest
import torch

import tlsgen
from oracle import exact, rqi

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def T():
    from paper_2305_19028_b200 import tlsrqi
    tlsrqi.lib()
    return tlsrqi


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


@pytest.mark.parametrize("fmt", ["fp16", "bf16", "fp32", "fp64"])
@pytest.mark.parametrize("n", [20, 96, 512, 1000, 2048])
def test_apply_through_inverse(T, fmt, n):
    """P^{-1} y and P^{-T} y through the GPU's W against the oracle's substitutions, to
    the inverse's accuracy kappa(R~) u (W is formed from R~, so the maps agree)."""
    rng = np.random.default_rng(n)
    A = rng.standard_normal((4 * n, n)) * np.logspace(0, -2, n)[None, :]
    pc = rqi.factor_precond(A, fmt)
    R = T.tls_precond_import(pc.Rt, pc.d, pc.normA2, fmt)
    kap = np.linalg.cond(pc.Rt)
    Y = rng.standard_normal((2, n))
    for trans, f in ((0, rqi.apply_Pinv), (1, rqi.apply_PinvT)):
        got = T.tls_precond_apply(R, trans | 2, dev(Y)).cpu().numpy()
        for r in range(2):
            ref = f(pc, Y[r])
            assert _rel(got[r], ref) <= 20 * kap * 2.0 ** -53, (trans, r)


@pytest.mark.parametrize("name,fmt", [("cfg1", "fp16"), ("cfg1", "bf16"), ("cfg2w", "fp16"), ("cfg2w", "bf16"),
                                      ("cfg2w", "fp32"), ("vanhuffel", "fp16"), ("random", "bf16")])
def test_rqi_parity_inverse(T, name, fmt):
    """Whole solve with precond_apply = 2 on the oracle's R~: status, termination, RQI
    count, PCG counts +-2; x to 1e-9 and sigma to 1e-12 against the oracle's inverse run
    and the SVD."""
    P = tlsgen.config(name) if name.startswith("cfg") else tlsgen.paper_problem(name)
    pc = rqi.factor_precond(P.A, fmt)
    res = rqi.rqi_pcgtls_mp(P.A, P.b, pc, opts=rqi.RqiOptions(precond_apply=2))
    R = T.tls_precond_import(pc.Rt, pc.d, pc.normA2, fmt)
    M = T.matrix(T.dense_operand(dev(P.A)), n=P.n)
    rc, x, sig, info = T.tls_rqi_pcgtls(M, dev(P.b), R, opts=T.tls_rqi_opts_default(precond_apply=2))
    assert info["status"] == res.status == rqi.OK
    assert info["termination"] == res.termination and info["rqi_iters"] == res.rqi_iters
    for a, b in zip(info["pcg_iters"], res.pcg_iters):
        assert abs(a[0] - b[0]) <= 2 and abs(a[1] - b[1]) <= 2
    ex = exact.tls_svd(P.A, P.b)
    x = x.cpu().numpy()
    assert _rel(x, res.x) <= 1e-9 and _rel(x, ex.x) <= 1e-9
    assert abs(sig - res.sigma) / res.sigma <= 1e-12 and abs(sig - ex.sigma) / ex.sigma <= 1e-11


def test_inverse_csr_and_wide(T):
    """CSR cfg3-small and a 6144 x 1536 dense problem through the GPU's own factorization:
    the inverse and the substitution solves agree (status, RQI count, x, sigma)."""
    P = tlsgen.config("cfg3", m=20000, n=500)
    M = T.matrix_csr(torch.as_tensor(P.rowptr, device="cuda"), torch.as_tensor(P.colidx, device="cuda"),
                     torch.as_tensor(P.vals, device="cuda"), P.n)
    D = tlsgen.dense_problem(6144, 1536, 1e3, 1e-3, 11, twin=True)
    for M_, b in ((M, torch.as_tensor(P.b, device="cuda")), (T.matrix(dev(D.A)), dev(D.b))):
        rc, R, _ = T.tls_factor_precond(M_, "fp16")
        assert rc == 0
        rc, x1, s1, i1 = T.tls_rqi_pcgtls(M_, b, R, opts=T.tls_rqi_opts_default(precond_apply=1))
        rc, x2, s2, i2 = T.tls_rqi_pcgtls(M_, b, R, opts=T.tls_rqi_opts_default(precond_apply=2))
        assert i1["status"] == i2["status"] == 0 and i1["rqi_iters"] == i2["rqi_iters"]
        assert _rel(x2.cpu().numpy(), x1.cpu().numpy()) <= 1e-9
        assert abs(s2 - s1) / s1 <= 1e-12
        # and against the oracle's explicit-inverse run on the same R~ (not only GPU vs GPU)
        Rt, d, nrm = T.tls_precond_export(R)
        if M_ is M:
            import scipy.sparse
            A_h = scipy.sparse.csr_matrix((P.vals, P.colidx, P.rowptr), shape=(P.m, P.n))
            b_h = P.b
        else:
            A_h, b_h = D.A, D.b
        res = rqi.rqi_pcgtls_mp(A_h, b_h, rqi.Precond(Rt, d, "fp16", nrm), opts=rqi.RqiOptions(precond_apply=2))
        assert i2["status"] == res.status and i2["rqi_iters"] == res.rqi_iters
        assert [tuple(p) for p in i2["pcg_iters"]] == [tuple(p) for p in res.pcg_iters]
        assert _rel(x2.cpu().numpy(), res.x) <= 1e-9
        assert abs(s2 - res.sigma) / res.sigma <= 1e-12
