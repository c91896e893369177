#!/bin/bash
# full GPU suite + smoke + the bench line after the k_gram_tc2 default
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 2700 python -m pytest -m gpu -q --timeout 1200 tests > gpurun_out/r02b_pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r02b_pytest_gpu.log | tail -10
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r02b_smoke.log
timeout -s KILL 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo bench rc=$?
cat gpurun_out/r02b_bench.json
