"""The pass sums' reduction + all-reduce as ONE kernel over peer memory (k_peer.cu, SURVEY §8(f)
NEXT-3).  On the real node every rank runs k_reduce_exchange on its own GPU and stores into the
others' buffers over NVLink; here (one GPU per call) it is checked two ways that never let
separate launches wait for each other (B200_PROFILING.md):
  - P emulated ranks in ONE cooperative launch (tls_peer_exchange_emulate): every rank's result is
    the rank-ordered sum of each rank's fixed-order reduction of its partial rows -- bit-exact
    against the same order evaluated on the host, identical on every rank, over repeated
    exchanges (the epoch-parity double buffers are reused);
  - the library path with a 1-rank communicator whose pass sums go through the exchange
    (tls_comm_peer_prepare / _connect): factor + solve bitwise identical to the same
    communicator without it.
"""
import uuid

import numpy as np
import pytest
import torch

import tlsgen

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def T():
    from paper_2305_19028_b200 import tlsrqi
    tlsrqi.lib()
    return tlsrqi


def _expected(parts):
    """Host evaluation in the kernel's order: per rank, 8 row groups summed in order, the group
    sums in order (k_reduce_partials); then the ranks' contributions in rank order 0..P-1."""
    P, G, W = parts.shape
    contrib = []
    for r in range(P):
        gs = []
        for grp in range(8):
            acc = np.zeros(W)
            for g in range(G * grp // 8, G * (grp + 1) // 8):
                acc = acc + parts[r, g]
            gs.append(acc)
        c = gs[0].copy()
        for k in range(1, 8):
            c = c + gs[k]
        contrib.append(c)
    tot = contrib[0].copy()
    for r in range(1, P):
        tot = tot + contrib[r]
    return tot


@pytest.mark.parametrize("P,G,W", [(1, 148, 2050), (2, 148, 2050), (3, 37, 1026), (8, 148, 4098), (4, 0, 70)])
def test_exchange_emulated_ranks(T, P, G, W):
    rng = np.random.default_rng(P * 1000 + W)
    parts = rng.standard_normal((P, G, W)) * np.exp2(rng.integers(-20, 20, (P, G, W)))
    out = T.tls_peer_exchange_emulate(torch.as_tensor(parts, device="cuda"), reps=5).cpu().numpy()
    exp = _expected(parts)
    for r in range(P):
        assert np.array_equal(out[r], exp), f"rank {r}"


def test_library_path_through_the_exchange_single_rank(T):
    """A 1-rank communicator with the peer exchange attached: every dense operator/residual pass
    ends with k_reduce_exchange instead of k_reduce_partials + the all-reduce; the factor and the
    solve (counts, x, sigma) are bitwise those of the same communicator without it."""
    P = tlsgen.config("cfg2w")
    A = torch.as_tensor(P.A, device="cuda")
    b = torch.as_tensor(P.b, device="cuda")
    n = P.A.shape[1]
    res = []
    for peer in (False, True):
        comm = T.tls_comm_init_shm(1, 0, f"/tls_peer_{uuid.uuid4().hex[:12]}", 0)
        try:
            if peer:
                rec = T.tls_comm_peer_prepare(comm, 2 * n + 2)
                T.tls_comm_peer_connect(comm, [rec])
            M = T.matrix(A)
            rc, R, fi = T.tls_factor_precond(M, "bf16", comm=comm)
            for pa in (1, 2):
                o = T.tls_rqi_opts_default(precond_apply=pa)
                rc, x, sig, info = T.tls_rqi_pcgtls(M, b, R, comm=comm, opts=o)
                res.append((peer, pa, x.cpu().numpy().view(np.uint64).copy(), sig, info["pcg_iters"], info["status"]))
        finally:
            T.tls_comm_destroy(comm)
    for a, b_ in zip(res[:2], res[2:]):
        assert a[1] == b_[1] and a[5] == b_[5] == 0
        assert np.array_equal(a[2], b_[2]) and a[3] == b_[3] and a[4] == b_[4]


def test_peer_capacity_too_small_is_refused(T):
    P = tlsgen.config("cfg1")
    A = torch.as_tensor(P.A, device="cuda")
    b = torch.as_tensor(P.b, device="cuda")
    comm = T.tls_comm_init_shm(1, 0, f"/tls_peer_{uuid.uuid4().hex[:12]}", 0)
    try:
        T.tls_comm_peer_connect(comm, [T.tls_comm_peer_prepare(comm, 8)])   # < 2n + 2
        M = T.matrix(A)
        with pytest.raises(T.TlsError):
            rc, R, fi = T.tls_factor_precond(M, "fp16", comm=comm)
            T.tls_rqi_pcgtls(M, b, R, comm=comm)
    finally:
        T.tls_comm_destroy(comm)


def test_precond_prepare_then_solve_allocates_nothing(T):
    """tls_precond_prepare makes the handle-owned buffers a solve would otherwise allocate on
    first use (the explicit inverse W, the fp32 copy of A): the solve then
    leaves the device's free memory unchanged, and gives the same bits as without prepare."""
    P = tlsgen.dense_problem(65536, 1024, 1e2, 1e-3, 5, twin=True, device="cuda", keep_factors=False)
    M = T.matrix(P.A)
    ws = T.workspace(M)
    o = T.tls_rqi_opts_default(precond_apply=2, u_p="fp32")
    rc, R0, _ = T.tls_factor_precond(M, "fp16", ws=ws)
    rc, x0, s0, i0 = T.tls_rqi_pcgtls(M, P.b, R0, opts=o, ws=ws)          # allocates W and the copy itself
    del R0
    rc, R, _ = T.tls_factor_precond(M, "fp16", ws=ws)
    T.tls_precond_prepare(M, R, 3, ws=ws)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    rc, x, s, info = T.tls_rqi_pcgtls(M, P.b, R, opts=o, ws=ws)
    torch.cuda.synchronize()
    assert torch.cuda.mem_get_info()[0] == free0
    assert info["status"] == i0["status"] == 0 and info["pcg_iters"] == i0["pcg_iters"]
    assert torch.equal(x, x0) and s == s0
    with pytest.raises(T.TlsError):
        T.tls_precond_prepare(M, R, 4, ws=ws)
