#!/bin/bash
# flush-cost experiment: the Gram kernels with the fp64 flush every 64 chunks (R11) vs only at the end
for tc in 256 128; do
  for sup in 64 1000000; do
    for epi in 2 0; do
      r=$(TLS_GRAM_SEGS=1 TLS_GRAM_TC=$tc TLS_GRAM_SUPER=$sup TLS_GRAM_EPI=$epi python tools/time_gram_tc2.py --one 1048576 1024 fp16 64 x 2>&1 | tail -1)
      echo "tc=$tc super=$sup epi=$epi: $r"
    done
  done
done
