"""Destination-row sharding for the multi-GPU path.

Host-side plumbing only (no method arithmetic): each of P ranks owns a
contiguous range of destination rows with ~m/P edges (binary search on
row_ptr), and the same range of X rows.  The local CSR keeps GLOBAL source
ids, so a rank's local fg_spmm / fg_sddmm runs unchanged on the all-gathered
X (fg_allgather_rows).  Per-row computation depends only on the row, so the
concatenated shard outputs are bit-identical to the 1-GPU output.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def nnz_balanced_offsets(row_ptr: np.ndarray, nranks: int) -> np.ndarray:
    """int64[nranks+1] row offsets; shard r = rows [off[r], off[r+1]) holding
    ~nnz/nranks edges (ties broken toward the lower row)."""
    row_ptr = np.asarray(row_ptr, np.int64)
    n = row_ptr.size - 1
    m = int(row_ptr[-1])
    off = np.empty(nranks + 1, np.int64)
    off[0], off[-1] = 0, n
    for r in range(1, nranks):
        target = (m * r) // nranks
        off[r] = int(np.searchsorted(row_ptr, target, side="left"))
    np.maximum.accumulate(off, out=off)
    off = np.minimum(off, n)
    return off


@dataclass
class Shard:
    rank: int
    nranks: int
    lo: int
    hi: int
    offsets: np.ndarray      # int64[nranks+1] vertex (row) ranges of all ranks
    row_ptr: np.ndarray      # local int64[hi-lo+1], rebased to 0
    col_idx: np.ndarray      # local int32[local nnz], GLOBAL source ids
    edge_lo: int             # global CSR position of the first local edge

    @property
    def n_local(self) -> int:
        return self.hi - self.lo

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])


def make_shard(row_ptr: np.ndarray, col_idx: np.ndarray, rank: int, nranks: int,
               offsets: np.ndarray | None = None) -> Shard:
    row_ptr = np.asarray(row_ptr, np.int64)
    off = nnz_balanced_offsets(row_ptr, nranks) if offsets is None else np.asarray(offsets, np.int64)
    lo, hi = int(off[rank]), int(off[rank + 1])
    e0, e1 = int(row_ptr[lo]), int(row_ptr[hi])
    return Shard(rank, nranks, lo, hi, off, row_ptr[lo:hi + 1] - e0, np.asarray(col_idx[e0:e1], np.int32), e0)
