#!/bin/bash
# why the explicit-inverse solve's passes are slower: PDL and the fused reduction on/off
python tools/prof_solve_split.py cfg4w 2>&1
echo "== TLS_PDL=0"; TLS_PDL=0 python tools/prof_solve_split.py cfg4w 2>&1
echo "== TLS_FUSE_REDUCE=0"; TLS_FUSE_REDUCE=0 python tools/prof_solve_split.py cfg4w 2>&1
echo "== TLS_PDL=0 TLS_FUSE_REDUCE=0"; TLS_PDL=0 TLS_FUSE_REDUCE=0 python tools/prof_solve_split.py cfg4w 2>&1
