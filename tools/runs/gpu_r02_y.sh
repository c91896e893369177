#!/bin/bash
# TRSV per-block timeline; fused-reduce bit test; PCG iteration timing
python tools/trsv_trace.py 1024 fp16 2>&1
python tools/trsv_trace.py 2048 fp16 2>&1 | head -3
python tools/time_trsv.py 2>&1 | head -8
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_reduce or graph_loop" 2>&1 | tail -3
python tools/time_pcg_iter.py --mode subst 2>&1
TLS_FUSE_REDUCE=0 python tools/time_pcg_iter.py --mode winv_fused 2>&1
python tools/time_pcg_iter.py --mode winv_fused 2>&1
