python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python tools/time_gram_fused.py > gpurun_out/gram_fused.log 2>&1; echo "rc=$?"; cat gpurun_out/gram_fused.log | tail -20
