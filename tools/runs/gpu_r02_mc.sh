#!/bin/bash
for segs in 1 8; do for mc in 0 1; do
  r=$(TLS_GRAM_SEGS=$segs TLS_GRAM_MC=$mc timeout 120 python tools/time_gram_tc2.py --one 1048576 1024 fp16 64 mc${mc}_s${segs} 2>&1 | tail -1)
  echo "segs=$segs mc=$mc: $r"
done; done
r=$(TLS_GRAM_MC=1 timeout 120 python tools/time_gram_tc2.py --one 200000 2000 fp16 64 mc1_b 2>&1 | tail -1); echo "200000x2000 mc=1: $r"
r=$(TLS_GRAM_MC=0 timeout 120 python tools/time_gram_tc2.py --one 200000 2000 fp16 64 mc0_b 2>&1 | tail -1); echo "200000x2000 mc=0: $r"
python -c "
import numpy as np
for a, b in (('mc0_s1', 'mc1_s1'), ('mc0_s8', 'mc1_s8')):
    x = np.load(f'/tmp/G_{a}_1048576_1024_fp16_64.npy'); y = np.load(f'/tmp/G_{b}_1048576_1024_fp16_64.npy')
    print(a, b, 'bit-identical', np.array_equal(x, y))
x = np.load('/tmp/G_mc0_b_200000_2000_fp16_64.npy'); y = np.load('/tmp/G_mc1_b_200000_2000_fp16_64.npy'); print('200000x2000 bit-identical', np.array_equal(x, y))
"
