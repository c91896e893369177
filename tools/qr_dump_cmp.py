"""Compare the GPU QR's working state after column J (TLS_QR_STOP/TLS_QR_DUMP, k_qr.cu) with the
oracle's state after the same step (a copy of oracle.qr.householder_qr_r's loop)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import rqi  # noqa: E402
from oracle.rounding import round_to  # noqa: E402
from paper_2305_19028_b200 import tlsrqi as T  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from qr_diff import problem  # noqa: E402


def oracle_state(A, fmt, J):
    rd = lambda x: round_to(np.asarray(x, dtype=np.float64), fmt)
    W = rd(np.array(A, dtype=np.float64))
    m, n = W.shape
    for j in range(J + 1):
        x = W[j:, j]
        sigma = float(rd(np.sqrt(rd(np.dot(x, x)))))
        alpha = -sigma if x[0] >= 0 else sigma
        v = x.copy()
        v[0] = float(rd(x[0] - alpha))
        vv = float(rd(np.dot(v, v)))
        beta = float(rd(2.0 / vv))
        wT = rd(beta * rd(v @ W[j:, j:]))
        W[j:, j:] = rd(W[j:, j:] - rd(np.outer(v, wT)))
        W[j, j] = alpha
        W[j + 1:, j] = 0.0
    return W, wT, (alpha, v[0], sigma, beta)


def main():
    m, n, fmt, J = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
    A = problem(m, n, 1e2, 1630)
    d, _ = rqi.norm_scaling(A)
    Wo, wTo, sc = oracle_state(A / d, fmt, J)
    path = "/tmp/qr_dump.bin"
    os.environ["TLS_QR_STOP"] = str(J)
    os.environ["TLS_QR_DUMP"] = path
    Ap = np.zeros((m, n + (n & 1)))
    Ap[:, :n] = A
    t = torch.as_tensor(Ap, device="cuda")
    try:
        T.tls_factor_precond_qr(T.matrix(t, n=n), fmt)
    except Exception as e:
        print("factor returned", e)
    raw = open(path, "rb").read()
    hdr = np.frombuffer(raw[:40], dtype=np.int64)
    mm, nn, ldw, nb, es = [int(v) for v in hdr]
    off = 40
    Wg = np.frombuffer(raw[off:off + mm * ldw * es], dtype=np.float32 if es == 4 else np.float64).reshape(mm, ldw)
    off += mm * ldw * es
    wTg = np.frombuffer(raw[off:off + nn * 8], dtype=np.float64); off += nn * 8
    scg = np.frombuffer(raw[off:off + 4 * nn * 8], dtype=np.float64).reshape(nn, 4); off += 4 * nn * 8
    P = np.frombuffer(raw[off:off + nb * nn * 8], dtype=np.float64).reshape(nb, nn)
    print("scalars gpu", scg[J].tolist(), "oracle", sc)
    wd = np.nonzero(wTg[J + 1:] != wTo[1:])[0] + J + 1
    print("wT differs at", len(wd), "cols, first", wd[:8].tolist())
    Wg = Wg[:, :nn].astype(np.float64)
    # trailing block rows > J, cols > J
    D = Wg[J + 1:, J + 1:] != Wo[J + 1:, J + 1:]
    r, c = np.nonzero(D)
    print("trailing W differs at", D.sum(), "entries; rows", np.unique(r + J + 1)[:10].tolist(), "cols",
          np.unique(c + J + 1)[:10].tolist())
    # next column's inner products from the partials vs the oracle's
    xn = Wo[J + 2:, J + 1]
    ip_or = xn @ Wo[J + 2:, J + 1:]
    ip_g = P.sum(axis=0)[J + 1:]
    bad = np.nonzero(np.abs(ip_g - ip_or) > 1e-12 * np.abs(xn) @ np.abs(Wo[J + 2:, J + 1:]))[0] + J + 1
    print("partials' inner products differ at", len(bad), "cols, first", bad[:10].tolist())


if __name__ == "__main__":
    main()
