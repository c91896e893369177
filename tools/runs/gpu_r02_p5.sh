#!/bin/bash
# PDL for k_reduce_partials and the substitution k_pcg_step; k_pcg_init loads batched
python tools/time_pcg_iter.py 2>&1 | grep '"pdl": true\|"graph": false'
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_gpu_csr.py tests/test_gpu_winv.py -q -x 2>&1 | tail -3
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02p5_bench.json 2> gpurun_out/r02p5_bench.err; echo bench rc=$?
TLS_PDL=0 timeout -s KILL 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-control > gpurun_out/r02p5_bench_nopdl.json 2> gpurun_out/r02p5_bench_nopdl.err; echo bench2 rc=$?
