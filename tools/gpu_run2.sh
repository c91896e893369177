set -x
timeout 300 python tools/time_trsv.py > gpurun_out/time_trsv.log 2>&1; echo trsv rc=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/time_trsv.log; tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json
