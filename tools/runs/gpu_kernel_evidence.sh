# ncu --set full of one launch of each remaining kernel family (the operator pass, the
# fp32 pass, the PCG step and the Cholesky are in gpu_round_measure.sh).
set -x
ncu_one() {  # name regex skip cmd...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 -o gpurun_out/ev_$name "$@" > /dev/null 2>&1; echo $name rc=$?
}
ncu_one round k_round_scaled 1 python tools/prof_gram.py
ncu_one gram_tc k_gram_tc 1 python tools/prof_gram.py
PROF_UF=fp64 PROF_M=65536 PROF_N=2048 ncu_one gram_f64 k_gram_f64 1 python tools/prof_gram.py
ncu_one colstats "k_pass<2, 2" 1 python tools/prof_gram.py
ncu_one csr_rows k_csr_rows 2 python tools/prof_csr.py
ncu_one csr_cols k_csr_cols 2 python tools/prof_csr.py
