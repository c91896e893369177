#!/bin/bash
# QR: blocked panel passes with one 4-column group per thread and 8 rows in flight
python tools/time_qr.py 4096x512 16384x1024 65536x2048 2>&1 | grep fp16
python tools/qr_blocked_check.py --time 2>&1 | grep "blocked:\|unblocked:\|identical"
timeout 1500 python -m pytest tests/test_gpu_qr.py tests/test_gpu_qr_blocked.py tests/test_gpu_multirank.py -q 2>&1 | tail -3
