# k_pass experiment: default build vs -DTLS_PASS_WIDE=1 (time_pass + ncu SM cycles of the 2-RHS operator pass)
for V in 0 1; do
  TLS_EXTRA_NVCC="-DTLS_PASS_WIDE=$V" python -m paper_2305_19028_b200.build --force > gpurun_out/build_$V.log 2>&1 || { cat gpurun_out/build_$V.log; exit 1; }
  echo "== TLS_PASS_WIDE=$V"
  timeout 300 python tools/time_pass.py 2>&1 | head -3
  timeout 300 ncu --metrics sm__cycles_elapsed.avg,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_pass -s 4 -c 1 python tools/prof_pass.py 2>&1 | grep -E "sm__cycles|duration|issue_active"
  timeout 600 python -m pytest -m gpu -q -x --timeout 600 tests/test_gpu_parity.py -k "pass or rqi_parity_imported" 2>&1 | tail -1
done
