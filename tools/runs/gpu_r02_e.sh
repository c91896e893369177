python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python tools/qr_diff.py > gpurun_out/qr_diff2.log 2>&1; cat gpurun_out/qr_diff2.log
timeout 600 python tools/time_qr.py > gpurun_out/time_qr.log 2>&1; cat gpurun_out/time_qr.log
timeout 1500 python -m pytest -m gpu -q --timeout 900 tests/test_gpu_qr.py tests/test_gpu_multirank.py > gpurun_out/pytest_e.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_e.log | tail -20
