"""Per-block timeline of the warp-specialised TRSV (TLS_TRSV_TRACE): for each solution block u
of one tls_precond_apply solve, when its owner warp entered solve() (its tile updates done),
when x_{u-1} arrived and when x_u was published (globaltimer, ns).  Prints the block period
(publish-to-publish), the owner's wait for x_{u-1} (positive: the chain is the limit) and the
arrival-to-publish time (the E product + the broadcast).  python tools/trsv_trace.py [n] [fmt]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
path = "/tmp/trsv_trace.txt"
os.environ["TLS_TRSV_TRACE"] = path
import numpy as np, torch
from paper_2305_19028_b200 import tlsrqi
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
fmt = sys.argv[2] if len(sys.argv) > 2 else "fp16"
rng = np.random.default_rng(0)
R = np.triu(rng.standard_normal((n, n))) / n
R[np.diag_indices(n)] = 1.0 + rng.random(n)
R = R.astype(np.float16).astype(np.float64)
pc = tlsrqi.tls_precond_import(R, np.ones(n), 1.0, fmt)
for trans, name in ((1, "forward (R^T)"), (0, "back (R)")):
    Y = torch.randn((1, n), dtype=torch.float64, device="cuda")
    for _ in range(3):
        tlsrqi.tls_precond_apply(pc, trans, Y)
    torch.cuda.synchronize()
    rows = np.array([[int(v) for v in l.split()] for l in open(path)], dtype=np.int64)
    rows = rows[np.argsort(rows[:, 2])]
    t0 = rows[:, 3].min()
    pub = rows[:, 5] - t0
    per = np.diff(pub)
    wait = (rows[1:, 4] - rows[1:, 3])
    a2p = (rows[1:, 5] - rows[1:, 4])
    print(f"n={n} {fmt} {name}: {len(rows)} blocks, first solve->last publish {pub[-1] - (rows[0, 3] - t0)} ns; "
          f"period mean {per.mean():.0f} ns (min {per.min()}, max {per.max()}); owner wait for x_(u-1) mean {wait.mean():.0f} ns "
          f"(<= 0 on {np.sum(wait <= 50)} blocks); arrival->publish mean {a2p.mean():.0f} ns")
    print("   u cta warp  solve  arrived  published (ns from the first solve)")
    for r in rows[:: max(1, len(rows) // 12)]:
        print(f"  {r[2]:3d} {r[0]:3d} {r[1]:4d} {r[3] - t0:6d} {r[4] - t0 if r[4] else 0:8d} {r[5] - t0:10d}")
