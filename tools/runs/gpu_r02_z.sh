# Round-2 closing evidence on the final code: GPU suite, smoke, bench cfg4w + cfg3, reference arm,
# launch list (host loop), ncu --set full of the operator pass.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest -m gpu -q --timeout 1200 tests > gpurun_out/r02f_pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r02f_pytest_gpu.log | tail -10
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r02f_smoke.log
timeout -s KILL 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02f_bench_cfg4w.json 2> gpurun_out/r02f_bench.err; echo bench rc=$?; cut -c1-400 gpurun_out/r02f_bench_cfg4w.json
timeout -s KILL 600 python bench.py --workload cfg3 --steps 20 --warmup 5 > gpurun_out/r02f_bench_cfg3.json 2> gpurun_out/r02f_bench_cfg3.err; echo cfg3 rc=$?
timeout -s KILL 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r02f_bench_reference_arm.json 2> gpurun_out/r02f_ref.err; echo ref rc=$?
TLS_PCG_GRAPH=0 BENCH_UNPROFILED=0 timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_launches_cfg4w.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-control > /dev/null 2>&1; echo ncu1 rc=$?
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:k_pass -s 2 -c 1 -o gpurun_out/r02f_k_pass_full python tools/prof_pass.py > /dev/null 2>&1; echo ncu2 rc=$?
