#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_qr_blocked.py -q -x > gpurun_out/pytest_qr_blocked.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_qr_blocked.log
python tools/qr_blocked_check.py --time > gpurun_out/qr_blocked.log 2>&1; echo "check rc=$?"
cat gpurun_out/qr_blocked.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/qrprof_blocked.csv \
    python tools/qr_blocked_prof.py blocked 16384 1024 > gpurun_out/qrprof_blocked.log 2>&1
python tools/qr_blocked_prof.py --summarize gpurun_out/qrprof_blocked.csv > gpurun_out/qrprof_blocked.txt 2>&1
head -12 gpurun_out/qrprof_blocked.txt
