python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python tools/qr_blocked_check.py --time > gpurun_out/qr_blocked.log 2>&1; echo rc=$?; cat gpurun_out/qr_blocked.log | tail -30
