# ncu --set full of every k_round_scaled / k_gram_tc2 launch of one factorization on HEAD
# (2^20 x 1024 fp16, default segments): per-launch time and DRAM bytes -> profiles/r02h_ncu_gram.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python tools/prof_gram.py; echo plain rc=$?
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k 'regex:k_round_scaled|k_gram_tc2|k_gram_reduce' -s 17 -c 17 -o gpurun_out/r02h_gram python tools/prof_gram.py > gpurun_out/r02h_ncu_gram.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/r02h_gram.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread > gpurun_out/r02h_gram_raw.csv 2>&1; echo csv rc=$?
