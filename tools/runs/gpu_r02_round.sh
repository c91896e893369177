# The Gram's rounding pass: three forms timed alone and beside the segmented SYRK, G compared;
# the Gram parity tests and the bench solve under the two new forms.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python tools/time_round.py > gpurun_out/r02f_round.log 2>&1; echo "time_round rc=$?"; cat gpurun_out/r02f_round.log
for RV in 2 ca; do
  TLS_ROUND=$RV timeout 900 python -m pytest -m gpu -q --timeout 600 tests/test_gpu_parity.py tests/test_gpu_stress.py -k "gram" > gpurun_out/r02f_pytest_round_$RV.log 2>&1; echo "pytest $RV rc=$?"; tail -2 gpurun_out/r02f_pytest_round_$RV.log
done
for RV in 1 2 ca; do
  TLS_ROUND=$RV timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-control > gpurun_out/r02f_bench_round_$RV.json 2> /dev/null; echo "bench $RV rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/r02f_bench_round_$RV.json'));print('$RV', d['ms_per_step'], d['kernel_share'].get('gram'), d.get('unprofiled',{}).get('tts_s'), d['clocks'])"
done
