# Standard box run: TRSV timing, GPU parity suite, 1-GPU bench (no e2e / cpu baseline unless FULL=1).
set -x
timeout 200 python tools/time_trsv.py 2>&1 | grep -E "nrhs=2" > gpurun_out/time_trsv.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
if [ "$FULL" = "1" ]; then EXTRA=""; else EXTRA="--no-e2e --no-cpu-baseline --no-control"; fi
timeout 600 python bench.py $EXTRA > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/time_trsv.log; tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
