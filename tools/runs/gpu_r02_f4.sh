#!/bin/bash
# CSR passes (8 gathers in flight, two row groups interleaved); explicit-inverse step loads batched
timeout 1500 python -m pytest tests/test_gpu_csr.py tests/test_gpu_winv.py tests/test_gpu_multirank.py tests/test_gpu_parity.py -q -x -k "csr or CSR or winv or multirank or fused or graph or cfg3 or options" 2>&1 | tail -3
python tools/time_pcg_iter.py 2>&1 | grep '"pdl": true'
python tools/prof_csr.py 2>&1 | tail -5
timeout -s KILL 600 python bench.py --workload cfg3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02f4_bench_cfg3.json 2> gpurun_out/r02f4_bench_cfg3.err; echo cfg3 rc=$?; tail -c 300 gpurun_out/r02f4_bench_cfg3.json
