python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python tools/qr_diff.py > gpurun_out/qr_diff.log 2>&1
TLS_QR_PDL=0 timeout 300 python tools/qr_diff.py >> gpurun_out/qr_diff.log 2>&1
TLS_QR_COOP=1 timeout 300 python tools/qr_diff.py >> gpurun_out/qr_diff.log 2>&1
cat gpurun_out/qr_diff.log
timeout 300 python tools/time_pcg_iter.py > gpurun_out/time_pcg_iter.log 2>&1; cat gpurun_out/time_pcg_iter.log
timeout 1200 python -m pytest -m gpu -q --timeout 900 tests/test_gpu_multirank.py tests/test_gpu_parity.py -k "multirank or minimality or fingerprint or sharded or winv or imported or end_to_end" > gpurun_out/pytest_c.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_c.log | tail -20
timeout 900 python -m pytest -m gpu -q --timeout 900 tests/test_gpu_winv.py > gpurun_out/pytest_c2.log 2>&1; echo "pytest winv rc=$?"; tail -3 gpurun_out/pytest_c2.log
