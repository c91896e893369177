#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/time_gram_tc2.py > gpurun_out/gram_tc2.log 2>&1; echo "time rc=$?"; cat gpurun_out/gram_tc2.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gram" > gpurun_out/pytest_gram_tc2.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gram_tc2.log
