"""Sustained (power-capped) bandwidth of the streaming passes: N back-to-back launches of
the fp64 operator pass (k_pass), the team-layout fp64 pass (TLS_PASS_TEAM), the fp32
pass, and a plain read (torch sum) over the same 8.6 GB, each timed with CUDA events,
with the SM clock sampled by nvidia-smi.  python tools/sustain.py [reps]"""
import os, subprocess, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_19028_b200 import tlsrqi as T

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
m, n = 1 << 20, 1024
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g)
q = torch.randn((2, n), dtype=torch.float64, device="cuda", generator=g)
M = T.matrix(A); ws = T.workspace(M)
R = T.tls_precond_import(torch.eye(n, dtype=torch.float64).numpy(), torch.ones(n, dtype=torch.float64).numpy(), 1.0, "fp64")
T.tls_pass_fp32(M, R, q, ws=ws)

def clocks(fn):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms", "100"],
                         stdout=subprocess.PIPE, text=True)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    time.sleep(0.2); p.terminate(); out, _ = p.communicate()
    v = [l.split(",") for l in out.strip().splitlines() if "," in l]
    sm = statistics.median(float(x[0]) for x in v) if v else float("nan")
    pw = statistics.median(float(x[1]) for x in v) if v else float("nan")
    return e0.elapsed_time(e1) / reps, sm, pw

for name, fn, by in (("k_pass op2 fp64", lambda: T.tls_pass(M, 0, q, ws=ws), 8.0 * m * n),
                     ("fp32 team pass", lambda: T.tls_pass_fp32(M, R, q, ws=ws), 4.0 * m * n),
                     ("torch A.sum(0) read", lambda: A.sum(0), 8.0 * m * n),
                     ("k_pass op2 fp64 (again)", lambda: T.tls_pass(M, 0, q, ws=ws), 8.0 * m * n)):
    fn(); torch.cuda.synchronize()
    ms, sm, pw = clocks(fn)
    print(f"{name:26s} {ms:.3f} ms  {by / ms / 1e9:.2f} TB/s  SM {sm:.0f} MHz  {pw:.0f} W", flush=True)
