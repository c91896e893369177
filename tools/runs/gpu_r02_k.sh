python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cond tools/micro/cond_graph.cu && /tmp/cond
timeout 600 python tools/time_pcg_iter.py > gpurun_out/time_pcg_iter2.log 2>&1; cat gpurun_out/time_pcg_iter2.log
timeout 2400 python -m pytest -m gpu -q --timeout 1200 tests > gpurun_out/pytest_k.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_k.log | tail -20
