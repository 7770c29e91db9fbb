"""Row sharding of A across GPUs (one process per GPU).

GPU g owns rows [r_g, r_{g+1}) chosen so every shard holds ~nnz/G nonzeros
(SURVEY 8e): the SpMM passes are bandwidth-bound per nonzero, so balancing
nonzeros balances time. Q is replicated; the per-shard partials
A_g^T (A_g Q) are summed by one NCCL all-reduce per iteration inside the native
library (comm.cu). Omega_g is rows [r_g, r_{g+1}) of the global sketch, so the
sharded solve draws the same Gaussian matrix as the single-GPU one.
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np

from .api import SparseMatrix


def shard_bounds(offsets: np.ndarray, world: int) -> List[int]:
    """Row boundaries r_0 = 0 <= r_1 <= ... <= r_G = rows balancing nonzeros."""
    rows = offsets.shape[0] - 1
    nnz = int(offsets[-1])
    if world < 1:
        raise ValueError("world size must be >= 1")
    bounds = [0]
    for g in range(1, world):
        bounds.append(int(np.searchsorted(offsets, nnz * g / world, side="left")))
    bounds.append(rows)
    for g in range(1, world + 1):  # monotone even with empty shards
        bounds[g] = max(bounds[g], bounds[g - 1])
    return bounds


def shard_rows(offsets: np.ndarray, world: int, rank: int) -> Tuple[int, int]:
    b = shard_bounds(offsets, world)
    return b[rank], b[rank + 1]


def shard_csr(a: SparseMatrix, r0: int, r1: int) -> SparseMatrix:
    """Rows [r0, r1) of a as a standalone CSR (column space unchanged)."""
    lo, hi = int(a.offsets[r0]), int(a.offsets[r1])
    return SparseMatrix(r1 - r0, a.cols, a.offsets[r0:r1 + 1] - lo, a.col_indices[lo:hi].copy(),
                        a.values[lo:hi].copy())
