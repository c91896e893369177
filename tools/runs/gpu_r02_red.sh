#!/bin/bash
python tools/time_pcg_iter.py > gpurun_out/time_pcg_iter5.log 2>&1; echo "pcg rc=$?"
python tools/time_peer.py > gpurun_out/time_peer2.log 2>&1; echo "peer rc=$?"; cat gpurun_out/time_peer2.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py tests/test_gpu_winv.py -q -x > gpurun_out/pytest_red.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_red.log
