python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python tools/time_gram_fused.py > gpurun_out/gram_fused.log 2>&1; cat gpurun_out/gram_fused.log
TLS_GRAM_FUSED=1 timeout 900 python -m pytest -m gpu -q --timeout 600 tests/test_gpu_parity.py -k "gram or factor_precond or end_to_end" > gpurun_out/pytest_i.log 2>&1; echo "fused pytest rc=$?"; tail -3 gpurun_out/pytest_i.log
