python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python tools/time_gram_fused.py --one 262144 1024 fp16 64 > /dev/null 2>&1
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:k_gram_fused -c 1 -o gpurun_out/fz_prof python tools/time_gram_fused.py --one 262144 1024 fp16 64 > gpurun_out/fz_ncu.log 2>&1
echo ncu rc=$?; tail -3 gpurun_out/fz_ncu.log
