python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -30
if [ "$REF" = "1" ]; then
  timeout 1200 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?"
  tail -3 gpurun_out/ref.err; cut -c1-600 gpurun_out/ref.json
fi
