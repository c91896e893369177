#!/bin/bash
for tc in 256 128; do for stg in 3 4; do for segs in 1 8; do
  [ $tc = 128 ] && [ $stg = 3 ] && continue
  r=$(TLS_GRAM_SEGS=$segs TLS_GRAM_TC=$tc TLS_GRAM_STAGES=$stg python tools/time_gram_tc2.py --one 1048576 1024 fp16 64 x 2>&1 | tail -1)
  echo "tc=$tc stages=$stg segs=$segs: $r"
done; done; done
r=$(TLS_GRAM_SEGS=1 TLS_GRAM_STAGES=3 TLS_GRAM_SUPER=1000000 python tools/time_gram_tc2.py --one 1048576 1024 fp16 64 x 2>&1 | tail -1)
echo "tc=256 stages=3 segs=1 no flush: $r"
