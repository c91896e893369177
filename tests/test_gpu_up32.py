"""GPU parity of the u_p = fp32 inner-solve operator (reading R23; SURVEY §8(f) NEXT-1;
PAPER.md:480-482) against oracle.rqi.operator_fp32 / RqiOptions(u_p="fp32").

The two sides accumulate in fp32 in different orders, so a pass is compared within
twice the closed-form fp32 bound around the exact product of the fp32 data; the solves
(whose outer loop is fp64) to the north_star tolerances."""
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


def _bounds(A, q):
    """Closed-form bound on |v - v_exact| and |s - s_exact| of the fp32 operator (both
    sides satisfy it, so their difference is within twice it)."""
    m, n = A.shape
    u = 2.0 ** -24
    g = lambda k: k * u / (1 - k * u)
    Ae = A.astype(np.float32).astype(np.float64)
    qe = q.astype(np.float32).astype(np.float64)
    t = Ae @ qe.T                                   # m x 2
    tb = g(n) * (np.abs(Ae) @ np.abs(qe).T)
    vb = g(m) * (np.abs(Ae).T @ (np.abs(t) + tb)) + np.abs(Ae).T @ tb
    sb = 2.0 * np.sum(np.abs(t) * tb, axis=0) + np.sum(tb * tb, axis=0)
    return (Ae.T @ t).T, vb.T, np.sum(t * t, axis=0), sb


@pytest.mark.parametrize("m,n", [(2, 1), (5, 3), (300, 37), (1000, 128), (4099, 200), (3000, 515), (20000, 1024),
                                 (2500, 1025), (3001, 2048)])
def test_pass_fp32_vs_oracle(T, m, n):
    """k_pass32 over every team layout (1-8 float4 per lane, one or two warps per row,
    several rows per slot for small n, ragged chunk tails) against operator_fp32."""
    rng = np.random.default_rng(m + 7 * n)
    A = rng.standard_normal((m, n)) * np.logspace(0, -1, n)[None, :]
    q = rng.standard_normal((2, n))
    Ad = T.dense_operand(dev(A))
    M = T.matrix(Ad, n=n)
    R = T.tls_precond_import(np.eye(n), np.ones(n), float(np.sum(A * A)), "fp64")
    v, s = T.tls_pass_fp32(M, R, dev(q))
    v, s = v.cpu().numpy(), s.cpu().numpy()
    v_ex, vb, s_ex, sb = _bounds(A, q)
    A32 = A.astype(np.float32)
    for r in range(2):
        tt, vo = rqi.operator_fp32(A32, q[r])
        assert np.all(np.abs(v[r] - v_ex[r]) <= vb[r] * 1.0001 + 1e-300)
        assert np.all(np.abs(v[r] - vo) <= 2.0 * vb[r] * 1.0001 + 1e-300)
        assert abs(s[r] - s_ex[r]) <= sb[r] * 1.0001 + 1e-300
        assert abs(s[r] - tt) <= 2.0 * sb[r] * 1.0001 + 1e-300


@pytest.mark.parametrize("name,fmt", [("cfg1", "fp16"), ("cfg1", "bf16"), ("cfg2w", "fp16"), ("cfg2w", "bf16"),
                                      ("cfg2w", "fp32"), ("random", "fp16"), ("vanhuffel", "bf16")])
def test_rqi_up_fp32_parity(T, name, fmt):
    """Whole solve with u_p = fp32 on the oracle's R~ (imported): status, termination and
    RQI count equal, PCG counts within +-2, x <= 1e-9 and sigma <= 1e-12 against the
    oracle's u_p = fp32 run and the SVD."""
    P = tlsgen.config(name) if name.startswith("cfg") else tlsgen.paper_problem(name)
    pc = rqi.factor_precond(P.A, fmt)
    res = rqi.rqi_pcgtls_mp(P.A, P.b, pc, opts=rqi.RqiOptions(u_p="fp32"))
    R = T.tls_precond_import(pc.Rt, pc.d, pc.normA2, fmt)
    M = T.matrix(T.dense_operand(dev(P.A)), n=P.n)
    rc, x, sig, info = T.tls_rqi_pcgtls(M, dev(P.b), R, opts=T.tls_rqi_opts_default(u_p="fp32"))
    assert info["status"] == res.status == rqi.OK
    assert info["termination"] == res.termination
    assert info["rqi_iters"] == res.rqi_iters
    for a, b in zip(info["pcg_iters"], res.pcg_iters):
        assert abs(a[0] - b[0]) <= 2 and abs(a[1] - b[1]) <= 2
    ex = exact.tls_svd(P.A, P.b)
    x = x.cpu().numpy()
    assert _rel(x, res.x) <= 1e-9 and _rel(x, ex.x) <= 1e-9
    assert abs(sig - res.sigma) / res.sigma <= 1e-12
    assert abs(sig - ex.sigma) / ex.sigma <= 1e-11


def test_up_fp32_wide_and_factor(T):
    """n = 1536 (two warps per row) through the GPU's own factorization: same status and
    RQI count as the u_p = fp64 solve on the same R~, and x/sigma agree with it."""
    P = tlsgen.dense_problem(8192, 1536, 1e3, 1e-3, 9, twin=True)
    M = T.matrix(dev(P.A))
    rc, R, _ = T.tls_factor_precond(M, "fp16")
    assert rc == 0
    rc, x64, s64, i64 = T.tls_rqi_pcgtls(M, dev(P.b), R)
    rc, x32, s32, i32 = T.tls_rqi_pcgtls(M, dev(P.b), R, opts=T.tls_rqi_opts_default(u_p="fp32"))
    assert i32["status"] == i64["status"] == 0
    assert i32["rqi_iters"] == i64["rqi_iters"]
    assert _rel(x32.cpu().numpy(), x64.cpu().numpy()) <= 1e-9
    assert abs(s32 - s64) / s64 <= 1e-12
    # and against the oracle's u_p = fp32 run on the same R~ (not only GPU vs GPU)
    Rt, d, nrm = T.tls_precond_export(R)
    res = rqi.rqi_pcgtls_mp(P.A, P.b, rqi.Precond(Rt, d, "fp16", nrm), opts=rqi.RqiOptions(u_p="fp32"))
    assert i32["status"] == res.status and i32["rqi_iters"] == res.rqi_iters
    for a, b in zip(i32["pcg_iters"], res.pcg_iters):
        assert abs(a[0] - b[0]) <= 2 and abs(a[1] - b[1]) <= 2
    assert _rel(x32.cpu().numpy(), res.x) <= 1e-9
    assert abs(s32 - res.sigma) / res.sigma <= 1e-12
