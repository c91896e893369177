#!/bin/bash
# register-column POTRF/TRSM (k_chol_dag): micro cycles, factorization time A/B, R~ bits, parity tests
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o /tmp/chol_reg tools/micro/chol_reg.cu && /tmp/chol_reg
for r in 1 0; do echo "== TLS_CHOL_REG=$r"; TLS_CHOL_REG=$r python tools/time_chol.py 2>&1 | tail -3; TLS_CHOL_REG=$r python tools/chol_trace.py 2000 2>&1 | head -6; done
for r in 0 1; do TLS_CHOL_REG=$r python -c "
import numpy as np, torch
from paper_2305_19028_b200 import tlsrqi as T
rng = np.random.default_rng(3)
A = torch.as_tensor(rng.standard_normal((8000, 2000)) * np.logspace(0, -2, 2000)[None, :], device='cuda')
M = T.matrix(A)
rc, R, _ = T.tls_factor_precond(M, 'fp16')
Rt, d, nrm = T.tls_precond_export(R)
np.save('/tmp/Rt_reg$r.npy', Rt)
"; done
python -c "
import numpy as np
a = np.load('/tmp/Rt_reg0.npy'); b = np.load('/tmp/Rt_reg1.npy')
print('R~ identical fraction between POTRF variants:', np.mean(a == b), 'max diff', np.max(np.abs(a-b)))
"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py -q -x -k "factor or chol or Chol or cholesky or breakdown" 2>&1 | tail -3
# inlined variant for comparison
TLS_EXTRA_NVCC=-DTLS_CHOL_REG_INLINE python -c "from paper_2305_19028_b200 import build; build.build(force=True)" && echo "== inlined" && python tools/time_chol.py 2>&1 | tail -3
