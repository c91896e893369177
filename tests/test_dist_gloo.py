"""Multi-GPU host logic on the CPU: world size 2 over torch.distributed (gloo).

The library's N > 1 path is: contiguous row shards
(paper_2305_19028_b200.dist.shard_rows), per-rank partial sums of every pass
over A, an fp64 all-reduce (sum; max for the column maxima), and replicated
n-vector work.  Here each rank computes its partials with the oracle's
primitives on its row block, all-reduces them with gloo, and the results must
equal the unsharded computation; the NCCL unique id is broadcast the way
dist.init_comm does it."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

import tlsgen
from oracle import rqi
from paper_2305_19028_b200.dist import broadcast_unique_id, shard_rows


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_rows_partition():
    for m in (1, 7, 200, 4096, 1 << 20, 65537):
        for P in (1, 2, 3, 4, 8):
            blocks = [shard_rows(m, P, r) for r in range(P)]
            assert blocks[0][0] == 0 and blocks[-1][1] == m
            for (lo, hi), (lo2, _) in zip(blocks, blocks[1:]):
                assert hi == lo2
            sizes = [hi - lo for lo, hi in blocks]
            assert max(sizes) - min(sizes) <= 1


def _allreduce(x: np.ndarray, op=tdist.ReduceOp.SUM) -> np.ndarray:
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    tdist.all_reduce(t, op=op)
    return t.numpy()


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        P = tlsgen.config("cfg1")
        A, b = P.A, P.b
        m, n = A.shape
        lo, hi = shard_rows(m, world, rank)
        Al, bl = A[lo:hi], b[lo:hi]
        res = {}
        # a1: column max (max-reduce) and sums of squares (sum-reduce) -> identical D
        cm = _allreduce(np.max(np.abs(Al), axis=0), tdist.ReduceOp.MAX)
        ss = _allreduce(np.sum(Al * Al, axis=0))
        d_full, nrm_full = rqi.column_scaling(A)
        _, E = np.frexp(cm)
        res["d_equal"] = bool(np.array_equal(np.ldexp(1.0, E - 1), d_full))
        res["normA2_rel"] = abs(ss.sum() - nrm_full) / nrm_full
        # a2: partial u_f Grams summed over ranks (chunks are local to each rank)
        G = _allreduce(rqi.gram_uf(Al, d_full, "fp16", 64))
        B = rqi.gram_exact_bound(A, d_full, "fp16", 64)
        Ah = rqi.round_to(A / d_full, "fp16")
        res["gram_in_bound"] = bool(np.all(np.abs(G - Ah.T @ Ah) <= 2 * B))
        # a7: operator pass, 2 RHS: v_r = sum_p A_p^T (A_p q_r), tau_r = sum_p ||A_p q_r||^2
        Q = np.random.default_rng(0).standard_normal((2, n))
        for r in range(2):
            t = Al @ Q[r]
            v = _allreduce(np.concatenate([Al.T @ t, [t @ t]]))
            tf = A @ Q[r]
            res[f"op_rel_{r}"] = np.linalg.norm(v[:n] - A.T @ tf) / np.linalg.norm(A.T @ tf)
            res[f"tau_rel_{r}"] = abs(v[n] - tf @ tf) / (tf @ tf)
        # a5: residual pass: v = A^T(b - Ax), rho = r^T r, gamma = b^T r
        x = np.random.default_rng(1).standard_normal(n)
        rl = bl - Al @ x
        v = _allreduce(np.concatenate([Al.T @ rl, [rl @ rl, bl @ rl]]))
        rf = b - A @ x
        res["resid_rel"] = np.linalg.norm(v[:n] - A.T @ rf) / np.linalg.norm(A.T @ rf)
        res["rho_rel"] = abs(v[n] - rf @ rf) / (rf @ rf)
        # replicated n-vector work: every rank derives identical bits from identical inputs
        sig2 = v[n] / (1 + x @ x)
        f = -v[:n] - sig2 * x
        allf = [torch.zeros(n, dtype=torch.float64) for _ in range(world)]
        tdist.all_gather(allf, torch.from_numpy(f))
        res["replicas_identical"] = all(torch.equal(allf[0], a) for a in allf)
        # NCCL unique id broadcast over the process group (dist.init_comm)
        uid = bytes(range(128)) if rank == 0 else None
        res["uid_ok"] = broadcast_unique_id(uid) == bytes(range(128))
        out[rank] = res
    finally:
        tdist.destroy_process_group()


def test_row_sharded_passes_world2():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for rank in range(world):
        r = out[rank]
        assert r["d_equal"] and r["gram_in_bound"] and r["replicas_identical"] and r["uid_ok"]
        assert r["normA2_rel"] < 1e-14
        for k in ("op_rel_0", "op_rel_1", "tau_rel_0", "tau_rel_1", "resid_rel", "rho_rel"):
            assert r[k] < 1e-13, (k, r[k])


class _LVec(np.ndarray):
    """A rank's rows of an m-vector: the inner product of two of them is all-reduced."""

    def __matmul__(self, other):
        return float(_allreduce(np.array([np.dot(np.asarray(self), np.asarray(other))]))[0])


def _solve_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        P = tlsgen.config("cfg2w", m=1024, n=96)
        A, b = P.A, P.b
        m, n = A.shape
        pc = rqi.factor_precond(A, "fp16")          # replicated factorization of the reduced Gram
        ref = rqi.rqi_pcgtls_mp(A, b, pc)
        lo, hi = shard_rows(m, world, rank)
        Al = np.ascontiguousarray(A[lo:hi])
        bl = np.ascontiguousarray(b[lo:hi]).view(_LVec)
        # the library's sharded structure: A q and b - A x stay local, A^T t and every
        # inner product of m-vectors are all-reduced, all n-vector work is replicated
        rqi.matvec = lambda _A, x: np.asarray(Al @ np.asarray(x)).view(_LVec)
        rqi.rmatvec = lambda _A, t: _allreduce(Al.T @ np.asarray(t))
        res = rqi.rqi_pcgtls_mp(Al, bl, pc)
        xs = [torch.zeros(n, dtype=torch.float64) for _ in range(world)]
        tdist.all_gather(xs, torch.from_numpy(np.asarray(res.x, dtype=np.float64)))
        out[rank] = {"same": (res.status, res.termination, res.rqi_iters, res.boot_iters, res.pcg_iters) ==
                             (ref.status, ref.termination, ref.rqi_iters, ref.boot_iters, ref.pcg_iters),
                     "x_rel": float(np.linalg.norm(res.x - ref.x) / np.linalg.norm(ref.x)),
                     "sig_rel": abs(res.sigma - ref.sigma) / ref.sigma,
                     "replicas": all(torch.equal(xs[0], v) for v in xs)}
    finally:
        tdist.destroy_process_group()


def test_row_sharded_solve_world2():
    """The whole RQI-PCGTLS-MP solve on two row shards over gloo (the N > 1 structure of
    SURVEY §8(e)) gives the unsharded oracle's status and counts, x and sigma to roundoff,
    and bit-identical x on both ranks."""
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_solve_worker, args=(world, port, out), nprocs=world, join=True)
    for rank in range(world):
        r = out[rank]
        assert r["same"] and r["replicas"]
        assert r["x_rel"] < 1e-12 and r["sig_rel"] < 1e-13


def _tsqr_worker(rank, world, port, out):
    """The exchange of the row-sharded QR preconditioner (tls_factor_precond_qr, R26): each
    rank factors its own rows (D from the all-reduced column sums of squares, R27; a column
    vanishing on a rank's rows takes the identity reflector, R26), writes its R into its
    rows of a zeroed (world n) x n stack (row i of rank p's R at stack row i world + p), the
    stack is sum-all-reduced (every other slot is zero, so the sum is exact), and every rank
    factors the stack."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.qr import householder_qr_r
        P = tlsgen.config("cfg1")
        A = P.A
        m, n = A.shape
        lo, hi = shard_rows(m, world, rank)
        c = _allreduce(np.sum(A[lo:hi] * A[lo:hi], axis=0))
        d = np.exp2(np.ceil((np.frexp(c)[1] - 1) / 2))                # 2^ceil(floor(log2 c) / 2)
        S = np.zeros((world * n, n))
        S[rank::world] = householder_qr_r(A[lo:hi] / d, "fp16", leaf=True)   # row-interleaved slots (R26)
        S = _allreduce(S)
        R = householder_qr_r(S, "fp16")
        pc = rqi.factor_precond_qr(A, "fp16", row_blocks=[shard_rows(m, world, r) for r in range(world)])
        allR = [torch.zeros(n * n, dtype=torch.float64) for _ in range(world)]
        tdist.all_gather(allR, torch.from_numpy(R.ravel().copy()))
        out[rank] = {"equal_oracle": bool(np.array_equal(R, pc.Rt)), "d_equal": bool(np.array_equal(d, pc.d)),
                     "replicas": all(np.array_equal(allR[0].numpy(), t.numpy()) for t in allR)}
    finally:
        tdist.destroy_process_group()


def test_row_sharded_qr_preconditioner_world2():
    """The TSQR exchange on two gloo ranks reproduces the oracle's TSQR with the shards as
    leaves bit for bit, identically on both ranks."""
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_tsqr_worker, args=(world, port, out), nprocs=world, join=True)
    for rank in range(world):
        r = out[rank]
        assert r["equal_oracle"] and r["d_equal"] and r["replicas"]


def _peer_attach_worker(rank, world, port, out):
    """Host logic of tlsrqi.comm_attach_peer (NEXT-3 peer exchange): every rank prepares its
    record, the records are all-gathered in rank order and each rank connects with the full,
    rank-ordered list (the C calls are stubbed: no GPU here)."""
    import os
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_19028_b200 import tlsrqi
        calls = []
        tlsrqi.tls_comm_peer_prepare = lambda comm, wcap: bytes([rank]) * 128
        tlsrqi.tls_comm_peer_connect = lambda comm, recs: calls.append(list(recs))
        tlsrqi.comm_attach_peer(1234, 2050)
        out[rank] = calls
    finally:
        tdist.destroy_process_group()


def test_peer_attach_gathers_records_in_rank_order_world2():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_peer_attach_worker, args=(world, port, out), nprocs=world, join=True)
    for rank in range(world):
        assert out[rank] == [[bytes([0]) * 128, bytes([1]) * 128]]
