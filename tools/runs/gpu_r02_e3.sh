#!/bin/bash
# explicit-inverse solve: does the cooperative step's SM footprint change the passes' time?
for c in 16 32 64 0; do echo "== TLS_WSTEP_CTAS=$c"; TLS_WSTEP_CTAS=$c python tools/prof_solve_split.py cfg4w 2>&1 | grep '"precond_apply": 2'; done
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv
