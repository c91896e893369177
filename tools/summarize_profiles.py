"""Copy a round's measurements from gpurun_out/ into profiles/ with text summaries:
bench line(s), config sweep, per-kernel launch summary of one bench step, ncu metrics
of the operator pass (traffic) and of a PCG step."""
import collections, csv, gzip, json, os, shutil, subprocess, sys

R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.environ.get("SUMMARY_SRC", os.path.join(R, "gpurun_out"))
P = os.path.join(R, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"

for src, dst in (("bench_full.json", f"{tag}_bench_cfg4w.json"), ("bench_cfg3.json", f"{tag}_bench_cfg3.json"),
                 ("configs.json", f"{tag}_configs.json")):
    if os.path.exists(os.path.join(G, src)):
        shutil.copy(os.path.join(G, src), os.path.join(P, dst))

# launch list -> per-kernel summary of this library's kernels (per step: total / 4 solves)
lc = os.path.join(G, "launches_cfg4w.csv")
if os.path.exists(lc):
    with open(lc, "rb") as fh, gzip.open(os.path.join(P, f"{tag}_bench_launches.csv.gz"), "wb") as out:
        out.write(fh.read())
    rows, h = [], None
    for r in csv.reader(open(lc)):
        if "Kernel Name" in r:
            h = r
            continue
        if h and len(r) == len(h):
            rows.append(r)
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    # steps in the capture = factorizations (one k_chol_dag launch each; bench.py runs warm-up,
    # timed, unprofiled and certificate solves)
    nsteps = max(1, sum(1 for r in rows if "k_chol_dag" in r[ki]))
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows:
        name = r[ki]
        if "tls::" not in name and "k_recip" not in name and "k_copy" not in name and "k_fill" not in name:
            continue
        k = name.split("(")[0].replace("void ", "").split("<")[0]
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui] == "ns" else (v * 1e3 if r[ui] == "ms" else v)
        tot[k] += v / nsteps
        cnt[k] += 1
    T = sum(tot.values())
    lines = ["# ncu --metrics gpu__time_duration.sum --clock-control none over `bench.py --steps 1 --warmup 3`:",
             f"# this library's kernels only, per step (total / {nsteps} factorizations), serialised and cold-cache per launch.",
             "# kernel                                   launches/step   us/step   share of kernel time"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{k:42s} {cnt[k] / nsteps:8.1f} {v:12.1f} {v / T * 100:7.2f}%")
    lines.append(f"{'total':42s} {sum(cnt.values()) / nsteps:8.1f} {T:12.1f}")
    open(os.path.join(P, f"{tag}_bench_launches_summary.txt"), "w").write("\n".join(lines) + "\n")


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return dict(zip(rows[0], rows[2] if len(rows) > 2 else rows[1]))


KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__cluster_dim_x", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg"]
for rep, dst, title in (("k_pass_full.ncu-rep", f"{tag}_ncu_k_pass_op2_full.txt",
                         "ncu --set full -k regex:k_pass -s 2 -c 1 python tools/prof_pass.py (2^20 x 1024, 2 RHS)"),
                        ("pcg_step.ncu-rep", f"{tag}_ncu_k_pcg_step.txt",
                         "ncu --set full -k regex:k_pcg_step -s 40 -c 1 (bench cfg4w, n=1024 fp16, 8-CTA cluster per RHS)"),
                        ("k_pass32_full.ncu-rep", f"{tag}_ncu_k_pass32_full.txt",
                         "ncu --set full -k regex:k_pass_team -s 2 -c 1 python tools/time_pass32.py (u_p = fp32 operator "
                         "pass, 2^20 x 1024 fp32 copy of A, 2 RHS; algorithmic 4.295 GB)"),
                        ("chol_full.ncu-rep", f"{tag}_ncu_k_chol_dag.txt",
                         "ncu --set full -k regex:k_chol_dag -s 1 -c 1 python tools/time_chol.py (tile-DAG Cholesky, n = 1024)")):
    path = os.path.join(G, rep)
    if not os.path.exists(path):
        continue
    shutil.copy(path, os.path.join(P, f"{tag}_{rep}"))
    d = ncu_raw(path)
    lines = [f"# {title}"] + [f"{k}: {d[k]}" for k in KEYS if k in d]
    for k, v in d.items():
        if "issue_stalled" in k and "per_issue_active" in k:
            try:
                if float(v) > 0.3:
                    lines.append(f"{k.replace('smsp__average_warps_issue_stalled_', 'stall ')}: {v}")
            except ValueError:
                pass
    open(os.path.join(P, dst), "w").write("\n".join(lines) + "\n")
    if rep.startswith("k_pass"):
        rd = float(d.get("dram__bytes_read.sum", "0").replace(",", ""))
        wr = float(d.get("dram__bytes_write.sum", "0").replace(",", ""))
        # ncu reports GB / MB in these columns for this report: normalise to bytes by unit row
        json.dump({"pass_op2_dram_bytes_per_launch": None, "ncu_dram_read": d.get("dram__bytes_read.sum"),
                   "ncu_dram_write": d.get("dram__bytes_write.sum"),
                   "source": f"profiles/{dst}"}, open(os.path.join(P, "traffic_ncu_raw.json"), "w"), indent=1)
print("ok")
