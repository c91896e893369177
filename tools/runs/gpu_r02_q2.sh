#!/bin/bash
# QR update pass with QD rows in flight per team; k_qr_fin with all partial rows in flight
for f in "-DTLS_QR_QD=1" "-DTLS_QR_QD=4" ""; do
  echo "== variant '$f'"
  TLS_EXTRA_NVCC="$f" python -c "from paper_2305_19028_b200 import build; build.build(force=True)" || exit 1
  python tools/time_qr.py 4096x512 16384x1024 65536x2048 2>&1 | grep fp16
  python tools/qr_blocked_check.py --time 2>&1 | grep "blocked:\|unblocked:"
done
timeout 1500 python -m pytest tests/test_gpu_qr.py tests/test_gpu_qr_blocked.py tests/test_gpu_multirank.py -q 2>&1 | tail -3
