"""Row sharding and the NCCL communicator for multi-GPU runs.

One process per GPU.  Every rank owns a contiguous row block of A and b; all
passes over A produce per-rank partial sums that the library all-reduces with
NCCL (ncclAllReduce, fp64) inside its host loop, so n-vectors stay replicated
and bit-identical on every rank.  torch.distributed is plumbing only: it
broadcasts NCCL's 128-byte unique id from rank 0.
"""
from __future__ import annotations

from typing import Tuple

import torch
import torch.distributed as tdist

from . import tlsrqi


def shard_rows(m: int, nranks: int, rank: int) -> Tuple[int, int]:
    """Contiguous row block [lo, hi) of `rank`; the first m % nranks ranks get one extra row."""
    if not (0 <= rank < nranks):
        raise ValueError("rank out of range")
    base, extra = divmod(m, nranks)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def shard_csr(rowptr, colidx, vals, lo: int, hi: int):
    """Rows [lo, hi) of a CSR matrix as a self-contained CSR block (rowptr rebased
    to 0); works on numpy arrays and torch tensors alike."""
    e0, e1 = int(rowptr[lo]), int(rowptr[hi])
    return rowptr[lo:hi + 1] - e0, colidx[e0:e1], vals[e0:e1]


def broadcast_unique_id(uid: bytes | None, group=None) -> bytes:
    """Rank 0's 128-byte id to every rank over the default process group."""
    obj = [uid if tdist.get_rank(group) == 0 else None]
    tdist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def init_comm(device: int, group=None):
    """NCCL communicator of the library for the current torch.distributed world
    (None when the world has one rank)."""
    world = tdist.get_world_size(group)
    if world == 1:
        return None
    rank = tdist.get_rank(group)
    uid = tlsrqi.tls_comm_get_unique_id() if rank == 0 else None
    uid = broadcast_unique_id(uid, group)
    return tlsrqi.tls_comm_init(world, rank, uid, device)


def local_matrix(A_local: torch.Tensor, m_global: int, row_offset: int):
    return tlsrqi.matrix(A_local, m_global=m_global, row_offset=row_offset)
