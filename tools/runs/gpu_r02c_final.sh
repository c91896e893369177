#!/bin/bash
# Round-2 final (after the blocked QR, the 128x256 Gram, the peer exchange): GPU test suite, smoke,
# the bench line, the reference arm (1 step), the cfg3 bench, the config sweep, the launch list
# (host loop: ncu does not see kernels inside conditional graph bodies), ncu --set full of the
# operator pass and of the Gram's SYRK.
mkdir -p gpurun_out/final
F=gpurun_out/final
python -c "import __graft_entry__ as g; g.build()" > $F/build.log 2>&1 || { cat $F/build.log; exit 1; }
timeout 2400 python -m pytest -m gpu -q --timeout 1200 tests > $F/r02c_pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" $F/r02c_pytest_gpu.log | tail -10
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $F/r02c_smoke.log 2>&1; echo smoke rc=$?; tail -1 $F/r02c_smoke.log
timeout -s KILL 1200 python bench.py --steps 20 --warmup 5 > $F/bench_full.json 2> $F/bench.err; echo bench rc=$?
timeout -s KILL 600 python bench.py --impl reference --steps 1 --warmup 1 > $F/bench_reference.json 2> $F/bench_reference.err; echo ref rc=$?
timeout -s KILL 600 python bench.py --workload cfg3 --steps 20 --warmup 5 > $F/bench_cfg3.json 2> $F/bench_cfg3.err; echo cfg3 rc=$?
timeout -s KILL 1200 python tools/run_configs.py --reps 3 --out $F/configs.json > $F/configs.log 2>&1; echo configs rc=$?
TLS_PCG_GRAPH=0 BENCH_UNPROFILED=0 timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/launches_cfg4w.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-control > /dev/null 2>&1; echo ncu1 rc=$?
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:k_pass -s 2 -c 1 -o $F/k_pass_full python tools/prof_pass.py > /dev/null 2>&1; echo ncu2 rc=$?
TLS_GRAM_SEGS=1 timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:k_gram_tc2 -c 1 -o $F/gram_tc2_full python tools/time_gram_tc2.py --one 1048576 1024 fp16 64 x > /dev/null 2>&1; echo ncu3 rc=$?
cat $F/bench_full.json | head -c 600; echo
