"""One table of ncu evidence per kernel family from the captured reports (gpurun_out/ or
profiles/): duration, DRAM bytes and % of peak, L2 %, the busiest pipe, issue activity.
  python tools/ncu_evidence.py > profiles/r01_ncu_kernel_evidence.txt"""
import csv, os, re, subprocess, sys
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REPS = [("k_pass<2,op> fp64 operator pass (a7)", "profiles/r01_k_pass_full.ncu-rep"),
        ("k_pass_team<float> u_p=fp32 operator pass", "profiles/r01_k_pass32_full.ncu-rep"),
        ("k_round_scaled (a2, fl_fp16(A D^-1))", "profiles/r01_k_round_scaled.ncu-rep"),
        ("k_gram_tc (a2, tcgen05 fp16 Gram)", "profiles/r01_k_gram_tc.ncu-rep"),
        ("k_gram_f64 (a2, DMMA fp64 Gram, 65536x2048)", "profiles/r01_k_gram_f64.ncu-rep"),
        ("k_chol_dag (a3, n=1024)", "profiles/r01_chol_full.ncu-rep"),
        ("k_pcg_step (a6+a8, 8-CTA cluster)", "profiles/r01_pcg_step.ncu-rep"),
        ("k_csr_rows (a7 CSR, cfg3)", "profiles/r01_k_csr_rows.ncu-rep"),
        ("k_csr_cols (a7 CSR, cfg3)", "profiles/r01_k_csr_cols.ncu-rep"),
        ("k_qr_step_v4 (NEXT-2 QR, 65536x2048, j=600)", "profiles/r01_ncu_qr_step_v4.ncu-rep")]
def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return {k: (u, v) for k, u, v in zip(rows[0], rows[1], rows[2])}
def num(d, k):
    u, v = d.get(k, ("", "nan"))
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return float("nan")
    return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}.get(u, 1)
print("# ncu --set full, one launch each (tools/runs/gpu_round_measure.sh, tools/runs/gpu_kernel_evidence.sh); the SM clock column")
print("# shows where ncu locked the base clock (1.1 GHz).  DRAM = dram__bytes_read+write; pipes = % of peak sustained active.")
print(f"{'kernel':46s} {'time':>9s} {'DRAM GB':>8s} {'DRAM%':>6s} {'L2%':>5s} {'tensor%':>8s} {'dmma%':>6s} {'fp64%':>6s} {'issue%':>7s} {'SM clk':>8s}")
for name, rel in REPS:
    path = os.path.join(R, rel)
    if not os.path.exists(path):
        continue
    d = raw(path)
    t = num(d, "gpu__time_duration.sum")
    by = num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum")
    cyc = num(d, "sm__cycles_elapsed.avg")
    print(f"{name:46s} {t * 1e3:7.3f}ms {by / 1e9:8.3f} {num(d, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} "
          f"{num(d, 'lts__throughput.avg.pct_of_peak_sustained_elapsed'):5.1f} "
          f"{num(d, 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'):8.1f} "
          f"{num(d, 'sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active'):6.1f} "
          f"{num(d, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):6.1f} "
          f"{num(d, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):7.1f} {cyc / t / 1e9 if t else 0:6.2f}GHz")
