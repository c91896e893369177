#!/bin/bash
for t in 0 1; do echo "== TLS_CHOL_TRSM=$t"; TLS_CHOL_TRSM=$t python tools/time_chol.py 2>&1 | tail -3; TLS_CHOL_TRSM=$t python tools/chol_trace.py 2000 2>&1 | head -6; done
python - <<'PY'
import numpy as np, torch, os, subprocess, sys
# bit-identity of R~ between the two TRSM layouts
from paper_2305_19028_b200 import tlsrqi as T
PY
for t in 0 1; do TLS_CHOL_TRSM=$t python -c "
import numpy as np, torch
from paper_2305_19028_b200 import tlsrqi as T
rng = np.random.default_rng(3)
A = torch.as_tensor(rng.standard_normal((8000, 2000)) * np.logspace(0, -2, 2000)[None, :], device='cuda')
M = T.matrix(A)
rc, R, _ = T.tls_factor_precond(M, 'fp16')
Rt, d, nrm = T.tls_precond_export(R)
np.save('/tmp/Rt_trsm$t.npy', Rt)
"; done
python -c "
import numpy as np
a = np.load('/tmp/Rt_trsm0.npy'); b = np.load('/tmp/Rt_trsm1.npy')
print('R~ bit-identical between TRSM layouts:', np.array_equal(a, b))
"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py -q -x -k "factor or chol or Chol or cholesky" 2>&1 | tail -2
