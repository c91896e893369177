python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for D in 0 1; do echo "== TLS_CHOL_DMMA=$D"; TLS_CHOL_DMMA=$D timeout 300 python tools/time_chol.py; done > gpurun_out/chol_dmma.log 2>&1; cat gpurun_out/chol_dmma.log
timeout 600 python tools/time_pcg_iter.py > gpurun_out/time_pcg_iter4.log 2>&1; cat gpurun_out/time_pcg_iter4.log | cut -c1-220
timeout 1500 python -m pytest -m gpu -q --timeout 900 tests/test_gpu_parity.py tests/test_gpu_stress.py -k "chol or factor or cfg4w or stress or bitwise or end_to_end or breakdown" > gpurun_out/pytest_o.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_o.log
