#!/bin/bash
TLS_GRAM_SEGS=1 TLS_GRAM_STAGES=3 ncu --set full --import-source on --clock-control none -k regex:k_gram_tc2 -c 1 -o gpurun_out/gram_tc2_full3 \
   python tools/time_gram_tc2.py --one 1048576 1024 fp16 64 x > gpurun_out/gram_tc2_full3.log 2>&1
echo "full rc=$?"
