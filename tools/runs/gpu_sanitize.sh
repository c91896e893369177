# compute-sanitizer over tools/sanitize_cases.py: memcheck, racecheck, synccheck, initcheck.
# Logs: gpurun_out/san_<tool>.log.  Each tool bounded by its own timeout.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/san_build.log 2>&1
timeout 300 python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1; echo plain rc=$?
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  timeout ${SAN_TIMEOUT:-900} $CS --tool $tool --target-processes all --print-limit 50 \
     python tools/sanitize_cases.py ${SAN_CASES} > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"
  tail -4 gpurun_out/san_$tool.log
done
