# Round-2 parity run: build, GPU test suite, full cfg5 sweep vs the oracle.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
nproc > gpurun_out/host_cores.txt; lscpu >> gpurun_out/host_cores.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
if [ "$CFG5" = "1" ]; then
  timeout 1800 python tools/cfg5_parity.py --out gpurun_out/r02_cfg5_parity.jsonl > gpurun_out/cfg5_parity.log 2>&1; echo "cfg5 rc=$?"
  tail -5 gpurun_out/cfg5_parity.log
fi
