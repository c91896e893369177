#!/usr/bin/env python
"""bench.py — TLS time-to-solution of the B200 RQI-PCGTLS-MP hot path.

One step = one whole hot path on one (A, b): tls_factor_precond (§8 rows a1-a3)
+ tls_rqi_pcgtls (a4-a9), inputs resident in HBM.  Default workload: cfg4w,
the well-posed twin of BASELINE.json configs[3] (dense 2^20 x 1024 fp64,
kappa 1e4, u_f fp16; reading R8), row-sharded over N GPUs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 is launched by torchrun (one process per GPU, RANK/LOCAL_RANK/WORLD_SIZE
from the env); times are CUDA events on the solve stream, max over ranks.
Rank 0 prints ONE JSON line.  `--impl reference` times the CPU oracle
(oracle/, the only reference this paper has): every step is one whole oracle
solve of the same workload on the host cores (no sample, no extrapolation).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "TLS time-to-solution (s) & PCG iters/s, % HBM roofline, 1/2/4/8 B200"
WORKLOADS = {
    # name: (tlsgen config, m, n, u_f, description)
    "cfg4w": ("cfg4w", 1 << 20, 1024, "fp16",
              "cfg4w: dense 1048576x1024 fp64 A=U diag(s) V^T, kappa 1e4, b noise 1e-3*N(0,1)/sqrt(m), u_f fp16"),
    "cfg4": ("cfg4", 1 << 20, 1024, "fp16",
             "cfg4 (literal): dense 1048576x1024 fp64, kappa 1e4, b noise 1e-3*N(0,1), u_f fp16"),
    "cfg2w": ("cfg2w", 4096, 512, "bf16", "cfg2w: dense 4096x512 fp64, kappa 1e3, u_f bf16"),
    "cfg5": ("cfg5:k1e4:e1e-6", 65536, 2048, "fp16", "cfg5 cell kappa 1e4 eps 1e-6: dense 65536x2048 fp64, u_f fp16"),
    "cfg3": ("cfg3", 200000, 2000, "fp16",
             "cfg3: CSR 200000x2000 fp64, 10 distinct uniform columns + column i mod 2000 per row, u_f fp16"),
}


def _env_int(k, d):
    v = os.environ.get(k)
    return int(v) if v not in (None, "") else d


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            j = json.load(fh)
        return float(j.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.p = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, smax, reasons = [], [], set()
        for ln in out.strip().splitlines():
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for name, val in zip(self.NAMES, f[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        loaded = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def make_problem(wl, device):
    import tlsgen
    cfg, m, n, u_f, _ = WORKLOADS[wl]
    if cfg == "cfg3":
        return tlsgen.config(cfg), u_f
    return tlsgen.config(cfg, device=device, keep_factors=False), u_f


# ----------------------------------------------------------------------------- oracle timing
def oracle_solve_timed(A_np, b_np, u_f):
    """The CPU oracle as it stands (oracle.rqi.solve: its scaling, fp32-chunked Gram, LAPACK
    Cholesky and RQI-PCGTLS-MP) timed end to end on the WHOLE workload on the host cores --
    no row sample, no extrapolation, the oracle's own iteration counts.  Returns
    (seconds, result, sample description, cores)."""
    from oracle import rqi as orq
    t0 = time.perf_counter()
    pc, res = orq.solve(A_np, b_np, u_f)
    t = time.perf_counter() - t0
    pcg = sum(a + b for a, b in res.pcg_iters)
    sample = (f"the whole oracle solve (oracle.rqi.solve: factor + RQI-PCGTLS-MP) on the full "
              f"{A_np.shape[0]}x{A_np.shape[1]} workload, unextrapolated, with the oracle's own counts "
              f"(status {res.status}, K={res.rqi_iters}, B0={res.boot_iters}, PCG={pcg}, {res.passes} passes over A)")
    return t, res, sample, orq._threads()


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle as it stands, on the host cores (rank 0 only): every
    warm-up and timed step is one whole oracle solve of the workload."""
    if rank != 0:
        return
    import torch
    wl = args.workload
    dev = "cuda:0" if torch.cuda.is_available() else "cpu"
    P, u_f = make_problem(wl, dev)
    if wl == "cfg3":
        import scipy.sparse
        A_np = scipy.sparse.csr_matrix((P.vals, P.colidx, P.rowptr), shape=(P.m, P.n))
        b_np = P.b
    else:
        A_np = P.A.cpu().numpy() if hasattr(P.A, "cpu") else P.A
        b_np = P.b.cpu().numpy() if hasattr(P.b, "cpu") else P.b
    del P
    if dev != "cpu":
        torch.cuda.empty_cache()
    times = []
    for it in range(args.warmup + args.steps):
        t, res, sample, cores = oracle_solve_timed(A_np, b_np, u_f)
        print(f"[reference] step {it}: {t:.2f} s", file=sys.stderr, flush=True)
        if it >= args.warmup:
            times.append(t)
    v = statistics.mean(times)
    line = {"metric": METRIC, "value": v, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": WORKLOADS[wl][4], "m": int(A_np.shape[0]), "n": int(A_np.shape[1]),
                       "u_f": u_f, "l2": "inputs larger than L2", "parallelism": "host cores"},
            "cpu_baseline": {"value": v, "unit": "s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "step_times_s": times, "status": int(res.status), "rqi_iters": res.rqi_iters,
            "boot_iters": res.boot_iters, "pcg_iters": [list(p) for p in res.pcg_iters]}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4w", choices=sorted(WORKLOADS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-control", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank, world, local = _env_int("RANK", 0), _env_int("WORLD_SIZE", 1), _env_int("LOCAL_RANK", 0)
    if args.gpus > 1 and world == 1:
        sys.exit("--gpus N > 1 must be launched with torchrun (one process per GPU)")

    import torch
    import torch.distributed as tdist
    if world > 1:
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.impl == "reference":
        run_reference(args, rank, world)
        if world > 1:
            tdist.destroy_process_group()
        return

    torch.cuda.set_device(local)
    from paper_2305_19028_b200 import build as _build, dist as pdist, tlsrqi
    _build.build()
    tlsrqi.lib()
    wl = args.workload
    _, m, n, u_f, desc = WORKLOADS[wl]

    P, u_f = make_problem(wl, f"cuda:{local}")
    m = P.m
    lo, hi = pdist.shard_rows(m, world, rank)
    csr = wl == "cfg3"
    keep_host = (rank == 0 and world == 1 and not args.no_cpu_baseline)
    if csr:
        import scipy.sparse
        rp, ci, va = pdist.shard_csr(P.rowptr, P.colidx, P.vals, lo, hi)
        dev = f"cuda:{local}"
        csr_t = (torch.as_tensor(rp, device=dev), torch.as_tensor(ci, device=dev), torch.as_tensor(va, device=dev))
        b_loc = torch.as_tensor(P.b[lo:hi], device=dev)
        A_loc = None
        A_full_host = scipy.sparse.csr_matrix((P.vals, P.colidx, P.rowptr), shape=(P.m, P.n)) if keep_host else None
        b_full_host = torch.as_tensor(P.b) if keep_host else None
        nnz_loc = int(va.size)
    else:
        A_loc = P.A[lo:hi].clone()
        b_loc = P.b[lo:hi].clone()
        A_full_host = P.A.cpu() if keep_host else None
        b_full_host = P.b.cpu() if keep_host else None
    del P
    torch.cuda.empty_cache()
    comm = pdist.init_comm(local) if world > 1 else None
    if csr:
        M = tlsrqi.matrix_csr(*csr_t, n, m_global=m, row_offset=lo)
    else:
        M = tlsrqi.matrix(A_loc, m_global=m, row_offset=lo)
    ws = tlsrqi.workspace(M)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        rc, R, fi = tlsrqi.tls_factor_precond(M, u_f, comm=comm, stream=stream, ws=ws)
        if R is None:
            raise RuntimeError(f"factor failed: {tlsrqi.STATUS.get(rc)}")
        rc, _, sig, info = tlsrqi.tls_rqi_pcgtls(M, b_loc, R, comm=comm, stream=stream, ws=ws, x_out=x)
        return fi, info, sig

    for _ in range(args.warmup):
        fi, info, sig = step()

    def timed():
        tlsrqi.tls_profile_enable(True)
        sampler = ClockSampler(local)
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        launches = 0
        passes = 0
        infos = []
        dbg = os.environ.get("BENCH_DEBUG") == "1"
        for _ in range(args.steps):
            if dbg:
                ev_a = torch.cuda.Event(enable_timing=True); ev_a.record(stream); th = time.perf_counter()
            fi, info, sig = step()
            if dbg:
                ev_b = torch.cuda.Event(enable_timing=True); ev_b.record(stream); ev_b.synchronize()
                print(f"[bench] step device {ev_a.elapsed_time(ev_b):.2f} ms host {1e3 * (time.perf_counter() - th):.2f} ms",
                      file=sys.stderr, flush=True)
            launches += fi["launches"] + info["launches"]
            passes += fi["passes"] + info["passes"]
            infos.append(info)
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            tdist.barrier()
        clocks = sampler.stop()
        prof = tlsrqi.tls_profile_read()
        tlsrqi.tls_profile_enable(False)
        ms_total = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            ms_total = float(t.item())
        return ms_total, launches, passes, infos, clocks, prof, sig

    # a run that saw hardware or thermal slowdown is measured once more (timing rules);
    # the decision is all-reduced so every rank repeats together
    BAD = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    ms_total, launches, passes, infos, clocks, prof, sig = timed()
    bad = 1.0 if BAD & set(clocks.get("reasons", [])) else 0.0
    if world > 1:
        t = torch.tensor([bad], dtype=torch.float64, device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        bad = float(t.item())
    if bad:
        first = clocks
        ms_total, launches, passes, infos, clocks, prof, sig = timed()
        clocks = dict(clocks, remeasured_after=first)
    ms_step = ms_total / args.steps
    tts = ms_step / 1e3

    # the same steps without the per-launch profiling events (the timed region above records two
    # CUDA events around every launch for the roofline): the PCG loops then run as the
    # graph-captured device-side loop (NEXT-3).  Reported beside `value`, not instead of it.
    unprof = None
    if os.environ.get("BENCH_UNPROFILED", "1") == "1":
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()
        u0 = torch.cuda.Event(enable_timing=True)
        u1 = torch.cuda.Event(enable_timing=True)
        u0.record(stream)
        for _ in range(args.steps):
            step()
        u1.record(stream)
        torch.cuda.synchronize()
        u_ms = u0.elapsed_time(u1)
        if world > 1:
            t = torch.tensor([u_ms], dtype=torch.float64, device="cuda")
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            u_ms = float(t.item())
        unprof = {"tts_s": u_ms / args.steps / 1e3, "pcg_loop": "CUDA graph (device-side WHILE)" if world == 1
                  else "host loop (multi-rank)", "note": "no per-launch profiling events"}

    info = infos[-1]
    pcg_per_solve = info["boot_iters"] + sum(a + b for a, b in info["pcg_iters"])
    a_passes = 3 + info["boot_iters"] + 1 + info["rqi_iters"] + sum(max(a, b) for a, b in info["pcg_iters"])
    peak, peak_kind = load_peaks()
    p2 = prof["pass_op2"]
    if csr:
        # row phase: rowptr, colidx, vals, t write (2 RHS); column phase: colptr, rowidx, vals,
        # t gathered once per nonzero (2 RHS) -- the operand is L2-resident (28 MB)
        ml = hi - lo
        bytes_per_pass = 8.0 * (ml + 1) + 12.0 * nnz_loc + 16.0 * ml + 8.0 * (n + 1) + 12.0 * nnz_loc + 16.0 * nnz_loc
    else:
        bytes_per_pass = 8.0 * (hi - lo) * M.ld
    roof = None
    if p2["count"] > 0:
        # 2-RHS operator launches that did work (the bootstrap CGLS also runs on the 2-RHS
        # kernel; launches issued after an early exit return at once and are not counted,
        # but their time stays in the denominator)
        working = args.steps * (info["boot_iters"] + sum(max(a, b) for a, b in info["pcg_iters"]))
        if csr:
            working = args.steps * sum(max(a, b) for a, b in info["pcg_iters"])
        working = max(1, min(working, p2["count"]))
        avg_ms = p2["ms"] / working
        ach = bytes_per_pass / (avg_ms * 1e-3) / 1e9
        # DRAM bytes per launch of this kernel from the committed `ncu --set full` capture of the
        # same launch (profiles/traffic_<workload>.json; ncu cannot run inside the timed region)
        traffic, traffic_src = None, None
        tpath = os.path.join(ROOT, "profiles", f"traffic_{wl}.json")
        if os.path.exists(tpath):
            with open(tpath) as fh:
                tj = json.load(fh)
            traffic = tj.get("pass_op2_dram_bytes_per_launch")
            traffic_src = f"committed ncu capture: profiles/traffic_{wl}.json ({tj.get('source', 'ncu --set full')})"
        roof = {"kernel": ("k_csr_rows<2,operator> + k_csr_cols<2> (t = A q, v = A^T t, 2 RHS; L2-resident operand)"
                           if csr else "k_pass<2,operator> (t = A q, v = A^T t, 2 RHS, one read of A)"),
                "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": traffic, "traffic_source": traffic_src, "algorithmic_bytes_per_launch": bytes_per_pass,
                "avg_launch_ms": avg_ms, "launches": p2["count"], "working_launches": working,
                "peak_kind": peak_kind}
    kshare = {k: v["ms"] / ms_total for k, v in prof.items() if v["count"]}
    # context for `frac`: a plain streaming read of the same operand (torch's column sum,
    # no arithmetic to speak of) timed right after the step loop, in the same clock /
    # power state; the copy-based peak of MEASURED_PEAKS.json is a short burst
    if roof is not None and not csr:
        A_loc.sum(0)
        torch.cuda.synchronize()
        r0 = torch.cuda.Event(enable_timing=True)
        r1 = torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        for _ in range(20):
            A_loc.sum(0)
        r1.record(stream)
        torch.cuda.synchronize()
        roof["plain_read_gbs_same_state"] = bytes_per_pass / (r0.elapsed_time(r1) / 20 * 1e-3) / 1e9
        roof["frac_of_plain_read"] = roof["achieved"] / roof["plain_read_gbs_same_state"]

    # ---- e2e: the same solve through tls_solve_host from pinned host buffers
    e2e = None
    if not args.no_e2e and not csr:
        A_h = A_loc.cpu().pin_memory()
        b_h = b_loc.cpu().pin_memory()
        x_h = torch.empty(n, dtype=torch.float64).pin_memory()
        dev_buf = torch.empty(tlsrqi.tls_solve_host_bytes(hi - lo, n, M.ld), dtype=torch.uint8, device="cuda")
        del A_loc
        torch.cuda.empty_cache()
        tlsrqi.tls_solve_host(A_h, b_h, u_f, dev_buf=dev_buf, stream=stream, x_host=x_h, comm=comm,
                              m_global=m, row_offset=lo)
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            tlsrqi.tls_solve_host(A_h, b_h, u_f, dev_buf=dev_buf, stream=stream, x_host=x_h, comm=comm,
                                  m_global=m, row_offset=lo)
        f1.record(stream)
        torch.cuda.synchronize()
        e_ms = f0.elapsed_time(f1)
        if world > 1:
            t = torch.tensor([e_ms], dtype=torch.float64, device="cuda")
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": e_ms / args.steps / 1e3, "unit": "s",
               "h2d_bytes_per_step": int(A_h.numel() * 8 + b_h.numel() * 8),
               "d2h_bytes_per_step": int(n * 8)}

    # the compensated certificate of the returned x (c2 step 8), one extra untimed solve
    rc_c, R_c, _ = tlsrqi.tls_factor_precond(M, u_f, comm=comm, stream=stream, ws=ws)
    sig_cert = None
    if R_c is not None:
        _, _, _, inf_c = tlsrqi.tls_rqi_pcgtls(M, b_loc, R_c, comm=comm, stream=stream, ws=ws, x_out=x,
                                               opts=tlsrqi.tls_rqi_opts_default(certify=1))
        sig_cert = inf_c["sigma_certified"]
        del R_c

    # TTS as a model: the step's passes over A at the HBM peak plus the
    # measured time of everything that is not a pass (Gram, Cholesky, PCG steps, ...)
    pass_cats = ("pass_op2", "pass_op1", "pass_resid", "colstats", "pass_op2_fp32", "reduce")
    non_pass_ms = sum(v["ms"] for k, v in prof.items() if k not in pass_cats) / args.steps
    passes_at_peak_ms = a_passes * bytes_per_pass / (peak * 1e9) * 1e3
    tts_model = {"a_passes": a_passes, "passes_at_peak_ms": passes_at_peak_ms,
                 "measured_non_pass_ms": non_pass_ms, "model_ms": passes_at_peak_ms + non_pass_ms,
                 "measured_ms": ms_step}

    # the uniform-precision control of the paper's comparison (SURVEY
    # §8(d)): the same solve with u_f = fp64 (exact R, fp64 Gram on CUDA cores), timed the
    # same way; its TTS over ours is the measured mixed-precision speedup on B200
    control = None
    if not args.no_control and world == 1 and not csr:
        def step64():
            rc, R, fi = tlsrqi.tls_factor_precond(M, "fp64", comm=comm, stream=stream, ws=ws)
            rc, _, sig, inf = tlsrqi.tls_rqi_pcgtls(M, b_loc, R, comm=comm, stream=stream, ws=ws, x_out=x)
            return inf
        step64()
        torch.cuda.synchronize()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(3):
            inf64 = step64()
        g1.record(stream)
        torch.cuda.synchronize()
        t64 = g0.elapsed_time(g1) / 3 / 1e3
        control = {"u_f": "fp64", "tts_s": t64, "status": inf64["status_name"], "rqi_iters": inf64["rqi_iters"],
                   "boot_iters": inf64["boot_iters"], "pcg_iters": inf64["pcg_iters"],
                   "measured_speedup_of_uf": t64 / tts}

    # the paper's experimental precision setting: the inner PCGTLS at
    # u_p = fp32 (R23), its operator pass on an fp32 copy of A (half the bytes); same
    # factorization, timed the same way as the line's value
    up32 = None
    if not args.no_control and not csr:
        o32 = tlsrqi.tls_rqi_opts_default(u_p="fp32")

        def step32():
            rc, R, fi = tlsrqi.tls_factor_precond(M, u_f, comm=comm, stream=stream, ws=ws)
            rc, _, sig, inf = tlsrqi.tls_rqi_pcgtls(M, b_loc, R, comm=comm, stream=stream, ws=ws, x_out=x, opts=o32)
            return inf, sig
        step32()
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()
        tlsrqi.tls_profile_enable(True)
        h0 = torch.cuda.Event(enable_timing=True)
        h1 = torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        for _ in range(args.steps):
            inf32, sig32 = step32()
        h1.record(stream)
        torch.cuda.synchronize()
        p32 = tlsrqi.tls_profile_read()["pass_op2_fp32"]
        tlsrqi.tls_profile_enable(False)
        t32 = h0.elapsed_time(h1) / args.steps
        if world > 1:
            t = torch.tensor([t32], dtype=torch.float64, device="cuda")
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            t32 = float(t.item())
        work32 = max(1, min(args.steps * sum(max(a, b) for a, b in inf32["pcg_iters"]), p32["count"]))
        avg32 = p32["ms"] / work32
        up32 = {"u_p": "fp32", "tts_s": t32 / 1e3, "status": inf32["status_name"],
                "rqi_iters": inf32["rqi_iters"], "boot_iters": inf32["boot_iters"], "pcg_iters": inf32["pcg_iters"],
                "sigma_rel_diff": abs(sig32 - sig) / sig, "speedup_vs_up_fp64": tts / (t32 / 1e3),
                "pass_fp32": {"kernel": "k_pass32 (u_p = fp32 operator pass, 4 m n bytes)",
                              "avg_launch_ms": avg32,
                              "achieved_gbs": 4.0 * (hi - lo) * n / (avg32 * 1e-3) / 1e9,
                              "frac": 4.0 * (hi - lo) * n / (avg32 * 1e-3) / 1e9 / peak}}

    # the explicit-inverse preconditioner application (R24; the default when sharded over
    # several ranks): same factorization, PCG steps on W = R~^{-1} over every SM
    winv = None
    if not args.no_control:
        ow = tlsrqi.tls_rqi_opts_default(precond_apply=2)

        def stepw():
            rc, R, fi = tlsrqi.tls_factor_precond(M, u_f, comm=comm, stream=stream, ws=ws)
            rc, _, sgw, inf = tlsrqi.tls_rqi_pcgtls(M, b_loc, R, comm=comm, stream=stream, ws=ws, x_out=x, opts=ow)
            return inf, sgw
        stepw()
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()
        tlsrqi.tls_profile_enable(True)
        k0 = torch.cuda.Event(enable_timing=True)
        k1 = torch.cuda.Event(enable_timing=True)
        k0.record(stream)
        for _ in range(args.steps):
            infw, sgw = stepw()
        k1.record(stream)
        torch.cuda.synchronize()
        pw = tlsrqi.tls_profile_read()
        tlsrqi.tls_profile_enable(False)
        tw = k0.elapsed_time(k1) / args.steps
        if world > 1:
            t = torch.tensor([tw], dtype=torch.float64, device="cuda")
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            tw = float(t.item())
        winv = {"precond_apply": "explicit inverse (R24)", "tts_s": tw / 1e3, "status": infw["status_name"],
                "rqi_iters": infw["rqi_iters"], "boot_iters": infw["boot_iters"], "pcg_iters": infw["pcg_iters"],
                "sigma_rel_diff": abs(sgw - sig) / sig, "speedup_vs_substitution": tts / (tw / 1e3),
                "pcg_step_us": 1e3 * pw["pcg_step"]["ms"] / max(1, pw["pcg_step"]["count"]),
                "pcg_step_us_substitution": 1e3 * prof["pcg_step"]["ms"] / max(1, prof["pcg_step"]["count"])}

    cpu = None
    if keep_host:
        import numpy as np
        t_cpu, res_cpu, sample, cores = oracle_solve_timed(A_full_host if csr else A_full_host.numpy(),
                                                           b_full_host.numpy(), u_f)
        cpu = {"value": t_cpu, "unit": "s", "cores": cores, "kind": "oracle", "sample": sample,
               "same_counts_as_gpu": (res_cpu.rqi_iters, [tuple(p) for p in res_cpu.pcg_iters]) ==
                                     (info["rqi_iters"], [tuple(p) for p in info["pcg_iters"]])}
        # the paper's flop model (oracle/perfmodel.py), "model only, no
        # hardware", at this (m, n, r = RQI steps): paper weights (u, u_p, u_q) = (fp64, fp32,
        # fp16) and the build's (fp64, fp64, u_f)
        from oracle import perfmodel
        cpu["paper_model_speedup"] = {
            "r": info["rqi_iters"],
            "paper_weights_fp64_fp32_fp16": perfmodel.speedup(m, n, info["rqi_iters"], "fp64", "fp32", "fp16"),
            "build_weights_fp64_fp64_uf": perfmodel.speedup(m, n, info["rqi_iters"], "fp64", "fp64", u_f)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": tts, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "m": m, "n": n, "u_f": u_f, "ld": int(M.ld),
                       "l2": ("operand L2-resident (CSR, %.0f MB)" % (20.0 * nnz_loc / 1e6) if csr else
                              "inputs larger than L2 (A = %.1f GB)" % (8.0 * m * n / 1e9)),
                       "parallelism": f"row-shard x{world} (NCCL all-reduce)"},
            "status": info["status_name"], "termination": info["termination_name"],
            "rqi_iters": info["rqi_iters"], "boot_iters": info["boot_iters"], "pcg_iters": info["pcg_iters"],
            "sigma": sig, "sigma_certified": sig_cert, "pcg_iters_per_s": pcg_per_solve / tts,
            # passes over A that do work: colstats + Gram read + setup + bootstrap CGLS + r_0
            # + one residual pass per RQI step + one batched operator pass per PCG iteration
            "a_passes_per_step": a_passes,
            "pass_launches_per_step": passes / args.steps,
            "a_passes_per_s": a_passes / tts,
            "roofline": roof, "kernel_share": kshare, "tts_model": tts_model,
            "gpu_launches": launches, "clocks": clocks, "e2e": e2e, "cpu_baseline": cpu,
            "uniform_fp64_control": control,
            "paper_precision_up_fp32": up32,
            "precond_inverse": winv,
            "unprofiled": unprof,
        }
        print(json.dumps(line), flush=True)
    if comm:
        tlsrqi.tls_comm_destroy(comm)
    if world > 1:
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
