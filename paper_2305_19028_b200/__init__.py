"""B200-native (sm_100a) hot path of RQI-PCGTLS-MP (Oktay & Carson, arXiv 2305.19028).

The numerical work runs in libtlsrqi.so (CUDA kernels behind the C ABI of
include/tlsrqi.h); `tlsrqi` is its ctypes binding, `dist` the row-sharding and
communicator plumbing over torch.distributed.
"""
from . import tlsrqi  # noqa: F401
from .tlsrqi import (  # noqa: F401
    PREC, STATUS, TERM, TlsError, Precond, matrix, dense_operand, workspace,
    lib,
)

__all__ = ["tlsrqi", "dist", "PREC", "STATUS", "TERM", "TlsError", "Precond", "matrix",
           "dense_operand", "workspace", "lib"]
