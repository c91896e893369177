# The 2-row rounding pass as the default: Gram tests (incl. the forms' bit-identity), the
# whole-path parity tests, smoke, the bench line.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest -m gpu -q --timeout 900 tests/test_gpu_stress.py tests/test_gpu_parity.py > gpurun_out/r02g_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02g_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r02g_smoke.log
timeout -s KILL 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02g_bench_cfg4w.json 2> gpurun_out/r02g_bench.err; echo bench rc=$?; cut -c1-300 gpurun_out/r02g_bench_cfg4w.json
