#!/bin/bash
# per-kernel times of the Gram (unsegmented) for both kernels, and one full capture of k_gram_tc2
mkdir -p gpurun_out
for tc in 256 128; do
  TLS_GRAM_SEGS=1 TLS_GRAM_TC=$tc ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv \
    --log-file gpurun_out/gram_tc${tc}_launches.csv python tools/time_gram_tc2.py --one 1048576 1024 fp16 64 x > /dev/null 2>&1
  echo "tc=$tc rc=$?"
  python tools/qr_blocked_prof.py --summarize gpurun_out/gram_tc${tc}_launches.csv
done
TLS_GRAM_SEGS=1 ncu --set full --import-source on --clock-control none -k regex:k_gram_tc2 -c 1 -o gpurun_out/gram_tc2_full \
   python tools/time_gram_tc2.py --one 1048576 1024 fp16 64 x > gpurun_out/gram_tc2_full.log 2>&1
echo "full rc=$?"
