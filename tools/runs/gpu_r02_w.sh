#!/bin/bash
# explicit-inverse PCG step: batched GEMV loads + merged block sums; fp64 DFMA latency micro
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_lat tools/micro/fp64_lat.cu && /tmp/fp64_lat
python tools/time_pcg_iter.py 2>&1
python tools/time_pcg_iter.py --n 2048 --m 8192 2>&1 | grep -v '"graph": false'
timeout 1200 python -m pytest tests/test_gpu_winv.py tests/test_gpu_multirank.py -q -x 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "graph_loop or nccl_path or options or precond_apply" 2>&1 | tail -3
