# Final check of HEAD after the opt-in k_round_bulk landed: full GPU test suite, smoke, bench (cfg4w).
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02i_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r02i_smoke.log
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02i_bench_cfg4w.json 2> gpurun_out/r02i_bench.err; echo bench rc=$?
timeout 1500 python -m pytest -m gpu -q --timeout 1200 tests > gpurun_out/r02i_pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r02i_pytest_gpu.log | tail -10
