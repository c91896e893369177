python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
TLS_FZ_PROF=1 timeout 300 python tools/time_gram_fused.py --one 1048576 1024 fp16 64 2>&1 | tail -3
TLS_FZ_PROF=1 timeout 300 python tools/time_gram_fused.py --one 65536 2048 fp16 64 2>&1 | tail -3
