# Round measurement: full bench line, all-config sweep, cfg3 bench, launch list of one bench step,
# ncu --set full of the operator pass (traffic) and of one 2-RHS PCG step.
set -x
timeout -s KILL 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench rc=$?
timeout -s KILL 900 python tools/run_configs.py --reps 3 > gpurun_out/configs.log 2>&1; echo configs rc=$?
timeout -s KILL 300 python bench.py --workload cfg3 > gpurun_out/bench_cfg3.json 2>/dev/null; echo cfg3 rc=$?
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4w.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-control > /dev/null 2>&1; echo ncu1 rc=$?
timeout -s KILL 300 ncu --set full --import-source on -k regex:k_pass -s 2 -c 1 -o gpurun_out/k_pass_full python tools/prof_pass.py > /dev/null 2>&1; echo ncu2 rc=$?
timeout -s KILL 300 ncu --set full --import-source on -k regex:k_pcg_step -s 40 -c 1 -o gpurun_out/pcg_step python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-control > /dev/null 2>&1; echo ncu3 rc=$?
timeout -s KILL 300 ncu --set full --import-source on -k regex:k_pass_team -s 2 -c 1 -o gpurun_out/k_pass32_full python tools/time_pass32.py 1048576 1024 2 > /dev/null 2>&1; echo ncu4 rc=$?
timeout -s KILL 300 ncu --set full --import-source on -k regex:k_chol_dag -s 1 -c 1 -o gpurun_out/chol_full python tools/time_chol.py > /dev/null 2>&1; echo ncu5 rc=$?
