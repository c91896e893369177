#!/bin/bash
# TRSV build-time variants, same box: default, E row preloaded, runs of 4 blocks per CTA, traced
for f in "" "-DTLS_TRSV_EPRE" "-DTLS_TRSV_RUN=4" "-DTLS_TRSV_RUN=2" "-DTLS_TRSV_TRACE" ""; do
  echo "== variant '$f'"
  TLS_EXTRA_NVCC="$f" python -c "from paper_2305_19028_b200 import build; build.build(force=True)" || exit 1
  python tools/time_trsv.py 2>&1 | grep "fp16" | grep "nrhs=1"
  python tools/time_pcg_iter.py --mode subst 2>&1
  if [ "$f" = "-DTLS_TRSV_TRACE" ]; then python tools/trsv_trace.py 1024 fp16 2>&1 | grep "^n="; python tools/trsv_trace.py 2048 fp16 2>&1 | grep "^n="; fi
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_gpu_winv.py -q 2>&1 | tail -4
