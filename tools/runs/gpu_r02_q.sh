#!/bin/bash
# blocked QR: GPU tests + per-kernel launch lists (blocked vs unblocked)
mkdir -p gpurun_out
python -m pytest tests/test_gpu_qr_blocked.py -q -x > gpurun_out/pytest_qr_blocked.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_qr_blocked.log
for kind in blocked unblocked; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/qrprof_$kind.csv \
    python tools/qr_blocked_prof.py $kind 16384 1024 > gpurun_out/qrprof_$kind.log 2>&1
  echo "ncu $kind rc=$?"
  python tools/qr_blocked_prof.py --summarize gpurun_out/qrprof_$kind.csv | head -20
done
