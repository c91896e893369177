#!/bin/bash
for segs in 1 8; do for ew in 8 16; do
  r=$(TLS_GRAM_SEGS=$segs TLS_GRAM_EW=$ew timeout 120 python tools/time_gram_tc2.py --one 1048576 1024 fp16 64 ew${ew}_s${segs} 2>&1 | tail -1)
  echo "segs=$segs ew=$ew: $r"
done; done
for ew in 8 16; do r=$(TLS_GRAM_EW=$ew timeout 120 python tools/time_gram_tc2.py --one 200000 2000 fp16 64 ew${ew}_b 2>&1 | tail -1); echo "200000x2000 ew=$ew: $r"; done
python -c "
import numpy as np
for a, b in (('ew8_s1', 'ew16_s1'), ('ew8_s8', 'ew16_s8')):
    x = np.load(f'/tmp/G_{a}_1048576_1024_fp16_64.npy'); y = np.load(f'/tmp/G_{b}_1048576_1024_fp16_64.npy')
    print(a, b, 'bit-identical', np.array_equal(x, y))
x = np.load('/tmp/G_ew8_b_200000_2000_fp16_64.npy'); y = np.load('/tmp/G_ew16_b_200000_2000_fp16_64.npy'); print('200000x2000 bit-identical', np.array_equal(x, y))
"
TLS_GRAM_SEGS=1 TLS_GRAM_EW=16 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_gram_tc2 -c 1 python tools/time_gram_tc2.py --one 1048576 1024 fp16 64 x 2>&1 | grep -i "duration\|k_gram" | head -4
TLS_GRAM_SEGS=1 TLS_GRAM_EW=8 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_gram_tc2 -c 1 python tools/time_gram_tc2.py --one 1048576 1024 fp16 64 x 2>&1 | grep -i "duration\|k_gram" | head -4
