# Round-2 closing evidence on HEAD: full GPU test suite, smoke, bench (cfg4w), reference arm, launch list.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest -m gpu -q --timeout 1200 tests > gpurun_out/r02h_pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r02h_pytest_gpu.log | tail -10
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r02h_smoke.log
timeout -s KILL 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02h_bench_cfg4w.json 2> gpurun_out/r02h_bench.err; echo bench rc=$?
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02h_bench_reference_arm.json 2> gpurun_out/r02h_bench_ref.err; echo ref rc=$?
TLS_PCG_GRAPH=0 BENCH_UNPROFILED=0 timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02h_launches_cfg4w.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-control > /dev/null 2>&1; echo ncu1 rc=$?
