#!/bin/bash
# substitution PCG step with the pass partials reduced inside k_pcg_step (NEXT-3)
python tools/time_pcg_iter.py 2>&1
python tools/time_pcg_iter.py --n 2048 --m 8192 2>&1 | grep '"pdl": true'
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_gpu_csr.py tests/test_gpu_up32.py -q -x 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 > gpurun_out/r02x_bench.json 2> gpurun_out/r02x_bench.err; tail -c 600 gpurun_out/r02x_bench.json
