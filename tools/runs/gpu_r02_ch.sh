#!/bin/bash
for bs in 16 32; do echo "== TLS_CHOL_BS=$bs"; TLS_CHOL_BS=$bs python tools/time_chol.py 2>&1 | tail -3; TLS_CHOL_BS=$bs python tools/chol_trace.py 2000 2>&1 | head -6; done
