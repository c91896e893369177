python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for S in 1 2 4 8; do for shape in "1048576 1024" "65536 2048"; do
  echo "segs=$S $shape: $(TLS_GRAM_SEGS=$S TLS_GRAM_FUSED=0 timeout 300 python tools/time_gram_fused.py --one $shape fp16 64 2>&1 | tail -1)"
done; done > gpurun_out/gram_segs.log 2>&1
cat gpurun_out/gram_segs.log
timeout 900 python -m pytest -m gpu -q --timeout 600 tests/test_gpu_parity.py -k "gram or factor_precond or end_to_end or cfg4w_full" > gpurun_out/pytest_j.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_j.log
