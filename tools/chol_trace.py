"""Critical-path analysis of the tile-DAG Cholesky (TLS_CHOL_TRACE): per step k the
POTRF(k), TRSM(k,k+1), UPDATE(k,k+1,k+1) wait/compute times, and per task type the
mean compute time.  python tools/chol_trace.py [n]"""
import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
path = "/tmp/chol_trace.txt"
os.environ["TLS_CHOL_TRACE"] = path
import numpy as np, torch
from paper_2305_19028_b200 import tlsrqi
rng = np.random.default_rng(0)
A = torch.as_tensor(rng.standard_normal((4 * n, n)), device="cuda")
M = tlsrqi.matrix(A)
ws = tlsrqi.workspace(M)
for _ in range(3):
    tlsrqi.tls_factor_precond(M, "fp16", ws=ws)
rows = [tuple(int(v) for v in l.split()) for l in open(path)]
t0 = min(r[4] for r in rows)
t1 = max(r[8] for r in rows)
print(f"n={n}: {len(rows)} tasks, kernel span {(t1 - t0) / 1e3:.1f} us")
byt = collections.defaultdict(list)
for r in rows:
    byt[r[0]].append(((r[6] - r[5]) / 1e3, (r[7] - r[6]) / 1e3, (r[8] - r[7]) / 1e3))
for ty, name in ((0, "POTRF"), (1, "TRSM"), (2, "UPDATE"), (3, "DIAG")):
    if ty not in byt:
        continue
    v = np.array(byt[ty])
    print(f"  {name:6s} n={len(v):5d} ready->2nd {v[:, 0].mean():6.2f}  ->computed {v[:, 1].mean():6.2f}  ->end {v[:, 2].mean():6.2f} us")
idx = {(r[0], r[1], r[2], r[3]): r for r in rows}
T = (n + 63) // 64
f = lambda x: (x - t0) / 1e3
print(" k | DIAG(k) = TRSM(k,k+1)+UPD+POTRF(k+1): start ready trsm-done+wait potrf-done end  (us)")
for k in range(0, T - 1):
    d = idx.get((3, k, 0, k + 1))
    if d:
        print(f"{k:2d} | {f(d[4]):7.1f} {f(d[5]):7.1f} {f(d[6]):7.1f} {f(d[7]):7.1f} {f(d[8]):7.1f}")
