python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python tools/time_pcg_iter.py > gpurun_out/time_pcg_iter3.log 2>&1; cat gpurun_out/time_pcg_iter3.log
timeout 2400 python -m pytest -m gpu -q -x --timeout 1200 tests > gpurun_out/pytest_l.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_l.log | tail -20
