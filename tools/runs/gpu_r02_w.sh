#!/bin/bash
mkdir -p gpurun_out
for tc in 256 128; do
  for sup in 64 1000000; do
    r=$(TLS_GRAM_SEGS=1 TLS_GRAM_TC=$tc TLS_GRAM_SUPER=$sup python tools/time_gram_tc2.py --one 1048576 1024 fp16 64 x 2>&1 | tail -1)
    echo "unsegmented tc=$tc super=$sup: $r"
  done
done
timeout 600 python tools/time_gram_tc2.py > gpurun_out/gram_tc2.log 2>&1; echo "time rc=$?"; cat gpurun_out/gram_tc2.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gram" > gpurun_out/pytest_gram_tc2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gram_tc2.log
