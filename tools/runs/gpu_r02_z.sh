#!/bin/bash
# TRSV: E row in registers before the wait, next owner first, runs of L blocks per CTA
for L in 1 2 4 8; do echo "== TLS_TRSV_RUN=$L"; TLS_TRSV_RUN=$L python tools/trsv_trace.py 1024 fp16 2>&1 | grep "^n="; TLS_TRSV_RUN=$L python tools/trsv_trace.py 2048 fp16 2>&1 | grep "^n="; TLS_TRSV_RUN=$L python tools/time_pcg_iter.py --mode subst 2>&1; done
python tools/time_trsv.py 2>&1 | head -16
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_gpu_winv.py -q -x 2>&1 | tail -3
