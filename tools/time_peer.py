"""Per-pass cost of the pass sums' reduction on one rank: k_reduce_partials (+ the all-reduce,
here a 1-rank shm communicator: a no-op copy) against k_reduce_exchange (the NEXT-3 peer
exchange attached to the same communicator), from the library's per-kernel profile of a solve
(category `reduce`), m x n = 262144 x 1024 dense, u_f fp16.  Also the emulated P = 8 exchange
(one cooperative launch of all 8 ranks' CTAs) timed over 200 exchanges.

  python tools/time_peer.py
"""
import os
import sys
import time
import uuid

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import tlsgen  # noqa: E402
from paper_2305_19028_b200 import tlsrqi as T  # noqa: E402

P = tlsgen.dense_problem(262144, 1024, 1e2, 1e-3, 3, twin=True, device="cuda", keep_factors=False)
M = T.matrix(P.A)
for peer in (False, True):
    comm = T.tls_comm_init_shm(1, 0, f"/tls_tp_{uuid.uuid4().hex[:10]}", 0)
    if peer:
        T.tls_comm_peer_connect(comm, [T.tls_comm_peer_prepare(comm, 2 * 1024 + 2)])
    rc, R, fi = T.tls_factor_precond(M, "fp16", comm=comm)
    T.tls_rqi_pcgtls(M, P.b, R, comm=comm)
    torch.cuda.synchronize()
    T.tls_profile_enable(True)
    rc, x, sig, info = T.tls_rqi_pcgtls(M, P.b, R, comm=comm)
    torch.cuda.synchronize()
    pr = T.tls_profile_read()
    T.tls_profile_enable(False)
    r = pr["reduce"]
    print(f"{'peer exchange' if peer else 'reduce + all-reduce'}: {1e3 * r['ms'] / max(1, r['count']):.1f} us per pass "
          f"({r['count']} passes), status {info['status']}, pcg {info['pcg_iters']}", flush=True)
    T.tls_comm_destroy(comm)
parts = torch.randn((8, 148, 2050), dtype=torch.float64, device="cuda")
T.tls_peer_exchange_emulate(parts, reps=10)
torch.cuda.synchronize()
for reps in (10, 210):
    t0 = time.perf_counter()
    T.tls_peer_exchange_emulate(parts, reps=reps)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    if reps == 10:
        t10 = t
print(f"emulated P = 8 (one launch for all ranks): {1e6 * (t - t10) / 200:.1f} us per exchange", flush=True)
