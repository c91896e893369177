#!/bin/bash
# QR: 4 rows ahead in the update pass, batched k_qr_fin loads, VtV prefetch in k_wy_T
python tools/time_qr.py 4096x512 16384x1024 65536x2048 2>&1 | grep fp16
python tools/qr_blocked_check.py --time 2>&1 | grep "blocked:\|unblocked:\|identical"
TLS_PCG_GRAPH=0 timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02q3_launches.csv python tools/qr_blocked_prof.py blocked 16384 1024 > /dev/null 2>&1; echo ncu rc=$?; python tools/qr_blocked_prof.py --summarize gpurun_out/r02q3_launches.csv
timeout 1500 python -m pytest tests/test_gpu_qr.py tests/test_gpu_qr_blocked.py tests/test_gpu_multirank.py -q 2>&1 | tail -3
