"""GPU parity of the blocked Householder QR in u_f with tensor-core WY trailing updates
(tls_factor_precond_qr_blocked; reading R29, SURVEY §8(f) NEXT-2 "on tensor cores") against
oracle.qr.householder_qr_r_blocked.

What is compared, and why not bit for bit: the panel steps round exactly as the oracle's (R25,
bit-identical when no trailing update happens, n <= 128); the trailing updates' sums -- V^T C and
V^T V in fp32 per 64-row chunk, V Y in fp32 -- are accumulated inside the tensor cores in an
implementation-defined order with truncation (R11), the oracle's in row order with
round-to-nearest, so the u_f results differ in the last place here and there and that
propagates like any rounding error of the factorization.  So:
  - D bit-exact; n <= 128 bit-identical to the oracle (R29 and R25 coincide there);
  - the GPU's R~ is as accurate a QR factor of fl(A D^-1) as the oracle's (Gram residual within
    1.5x of the oracle's), preconditions A as well (kappa(A P^-1) within 10%), and agrees with
    it normwise to a few u_f;
  - a solve with the GPU's blocked R~: the north_star tolerances against the oracle run on the
    same R~ (same status, termination, RQI and PCG counts; x 1e-9, sigma 1e-12) and the SVD.
"""
import numpy as np
import pytest
import torch

from oracle import exact, rqi
from oracle.qr import householder_qr_r_blocked
from oracle.rounding import round_to, unit_roundoff

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def T():
    from paper_2305_19028_b200 import tlsrqi
    tlsrqi.lib()
    return tlsrqi


def _problem(m, n, kappa, seed, spread=True):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((m, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)))
    A = (U * np.logspace(0, -np.log10(kappa), n)) @ V.T
    if spread:
        A = A * np.exp2(rng.integers(-4, 5, n))[None, :]
    x = rng.standard_normal(n)
    b = A @ x + 1e-3 * rng.standard_normal(m) * np.linalg.norm(A @ x) / np.sqrt(m)
    return A, b


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


@pytest.mark.parametrize("m,n,fmt", [(600, 128, "fp16"), (333, 47, "bf16")])
def test_one_panel_is_bit_identical(T, m, n, fmt):
    A, _ = _problem(m, n, 1e2, m + n)
    rc, R, _ = T.tls_factor_precond_qr_blocked(T.matrix(T.dense_operand(torch.as_tensor(A, device="cuda")), n=n), fmt)
    assert rc == 0
    Rt, d, nrm = T.tls_precond_export(R)
    pc = rqi.factor_precond_qr(A, fmt)
    assert np.array_equal(d, pc.d)
    assert np.array_equal(Rt, pc.Rt)
    assert np.array_equal(Rt, householder_qr_r_blocked(A / d, fmt, 128))


@pytest.mark.parametrize("m,n,fmt", [(1100, 530, "fp16"), (2048, 256, "bf16"), (3000, 700, "fp16"),
                                     (1500, 1000, "bf16")])
def test_blocked_vs_oracle_R29(T, m, n, fmt):
    A, _ = _problem(m, n, 1e2, m + n)
    rc, R, info = T.tls_factor_precond_qr_blocked(T.matrix(torch.as_tensor(A, device="cuda")), fmt)
    assert rc == 0
    Rt, d, nrm = T.tls_precond_export(R)
    d2, _ = rqi.norm_scaling(A)
    assert np.array_equal(d, d2)
    Ro = householder_qr_r_blocked(A / d, fmt, 128)
    Ah = round_to(A / d, fmt)
    G = Ah.T @ Ah
    assert np.linalg.norm(Rt.T @ Rt - G) <= 1.5 * np.linalg.norm(Ro.T @ Ro - G)
    u = unit_roundoff(fmt)
    assert _rel(Rt, Ro) <= 4 * u
    assert np.all(np.diag(Rt) > 0) and np.array_equal(np.tril(Rt, -1), np.zeros_like(Rt))
    assert np.array_equal(round_to(Rt, fmt), Rt)
    iu = np.triu_indices(n)
    assert np.mean(Rt[iu] == Ro[iu]) >= 0.3        # measured 0.57-0.93
    k_gpu = np.linalg.cond(A @ np.linalg.inv(Rt * d[None, :]))
    k_or = np.linalg.cond(A @ np.linalg.inv(Ro * d[None, :]))
    assert k_gpu == pytest.approx(k_or, rel=0.1)


@pytest.mark.parametrize("m,n,fmt", [(1100, 530, "fp16"), (4000, 300, "bf16")])
def test_blocked_solve_parity(T, m, n, fmt):
    A, b = _problem(m, n, 1e2, 7 * m + n, spread=False)
    M = T.matrix(torch.as_tensor(A, device="cuda"))
    rc, R, _ = T.tls_factor_precond_qr_blocked(M, fmt)
    assert rc == 0
    rc, x, sig, info = T.tls_rqi_pcgtls(M, torch.as_tensor(b, device="cuda"), R)
    Rt, d, nrm = T.tls_precond_export(R)
    res = rqi.rqi_pcgtls_mp(A, b, rqi.Precond(Rt, d, fmt, nrm))
    ex = exact.tls_svd(A, b)
    assert info["status"] == res.status == rqi.OK
    assert info["termination"] == res.termination and info["rqi_iters"] == res.rqi_iters
    assert info["pcg_iters"] == [tuple(p) for p in res.pcg_iters]
    assert _rel(x.cpu().numpy(), res.x) <= 1e-9 and _rel(x.cpu().numpy(), ex.x) <= 1e-9
    assert abs(sig - res.sigma) / res.sigma <= 1e-12


def test_blocked_refuses(T):
    A, _ = _problem(300, 40, 10.0, 1)
    M = T.matrix(torch.as_tensor(A, device="cuda"))
    for fmt in ("fp32", "fp64"):
        with pytest.raises(T.TlsError):
            T.tls_factor_precond_qr_blocked(M, fmt)
