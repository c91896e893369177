"""SM clock and power while cfg4w solves run back to back, substitution vs explicit inverse
(nvidia-smi sampled every ~20 ms in a thread during ~3 s of each).  python tools/clock_split.py"""
import os, sys, subprocess, threading, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import tlsgen
from paper_2305_19028_b200 import tlsrqi as T
torch.cuda.set_device(0)
P = tlsgen.config("cfg4w", device="cuda", keep_factors=False)
M = T.matrix(P.A)
ws = T.workspace(M)
rc, R, _ = T.tls_factor_precond(M, "fp16", ws=ws)


def sample(stop, out):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True).stdout.strip().split(",")
        try:
            out.append((float(r[0]), float(r[1])))
        except (ValueError, IndexError):
            pass
        time.sleep(0.02)


for rep in range(2):
    for pa in (1, 2):
        o = T.tls_rqi_opts_default(precond_apply=pa)
        T.tls_rqi_pcgtls(M, P.b, R, opts=o, ws=ws)
        torch.cuda.synchronize()
        stop, out = threading.Event(), []
        th = threading.Thread(target=sample, args=(stop, out))
        th.start()
        t0 = time.time()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        k = 0
        while time.time() - t0 < 3.0:
            T.tls_rqi_pcgtls(M, P.b, R, opts=o, ws=ws)
            k += 1
        e1.record()
        torch.cuda.synchronize()
        stop.set()
        th.join()
        clk = [c for c, _ in out]
        pw = [p for _, p in out]
        print(f"precond_apply={pa}: {e0.elapsed_time(e1) / k:.2f} ms per solve over {k} solves; "
              f"SM clock median {statistics.median(clk):.0f} MHz (min {min(clk):.0f}), power median {statistics.median(pw):.0f} W "
              f"({len(out)} samples)", flush=True)
