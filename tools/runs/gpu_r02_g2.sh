#!/bin/bash
# the Gram changes since the last full run: stress + parity Gram tests, QR blocked (atb path), smoke
timeout 1500 python -m pytest tests/test_gpu_stress.py tests/test_gpu_parity.py tests/test_gpu_qr_blocked.py -q -x -k "gram or Gram or blocked or one_panel or refuses" > gpurun_out/pytest_gram2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gram2.log
timeout 600 python tools/time_gram_tc2.py > gpurun_out/gram_tc2_final.log 2>&1; cat gpurun_out/gram_tc2_final.log
