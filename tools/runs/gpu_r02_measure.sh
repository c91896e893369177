# Round-2 measurement: smoke, the bench line as the driver runs it, the reference arm, the launch
# list of one bench step, and ncu --set full of the operator pass (traffic).
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/r02_smoke.log
timeout -s KILL 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo bench rc=$?
tail -2 gpurun_out/r02_bench.err; cut -c1-400 gpurun_out/r02_bench.json
timeout -s KILL 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02_ref.json 2> gpurun_out/r02_ref.err; echo ref rc=$?
cut -c1-300 gpurun_out/r02_ref.json
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg4w.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-control > /dev/null 2>&1; echo ncu1 rc=$?
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:k_pass -s 2 -c 1 -o gpurun_out/r02_k_pass_full python tools/prof_pass.py > /dev/null 2>&1; echo ncu2 rc=$?
