#!/bin/bash
# Gram split reduction with (tile, 8-row) CTAs; fingerprint sum on one warp
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "gram or factor or fingerprint or cfg4w or chol" 2>&1 | tail -3
python tools/time_chol.py 2>&1 | tail -3
TLS_PCG_GRAPH=0 BENCH_UNPROFILED=0 timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02g3_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-control > /dev/null 2>&1; echo ncu rc=$?
