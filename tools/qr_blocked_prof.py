"""One QR factorization (blocked R29 or unblocked R25) for an ncu launch list:
  ncu --metrics gpu__time_duration.sum --csv python tools/qr_blocked_prof.py blocked 16384 1024
and the per-kernel-name summary of such a list:
  python tools/qr_blocked_prof.py --summarize launches.csv
"""
import csv
import re
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def summarize(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(anonymous namespace\)::|<unnamed>::", "", r[ik]).replace("void ", "")
        name = re.split(r"[<(]", name)[0]
        tot[name] += float(r[iv].replace(",", "")) * 1e-6   # ns -> ms
        cnt[name] += 1
    s = sum(tot.values())
    for k in sorted(tot, key=tot.get, reverse=True):
        print(f"{k:32s} {cnt[k]:6d} launches {tot[k]:9.3f} ms  {100 * tot[k] / s:5.1f}%")
    print(f"{'total':32s} {sum(cnt.values()):6d} launches {s:9.3f} ms")


def main():
    if sys.argv[1] == "--summarize":
        summarize(sys.argv[2])
        return
    import torch
    from paper_2305_19028_b200 import tlsrqi as T
    kind, m, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    A = torch.randn((m, n), dtype=torch.float64, device="cuda")
    fn = T.tls_factor_precond_qr_blocked if kind == "blocked" else T.tls_factor_precond_qr
    rc, R, info = fn(T.matrix(A), "fp16")
    torch.cuda.synchronize()
    print(kind, m, n, rc, info["launches"])


if __name__ == "__main__":
    main()
