"""Test-only helpers: tiny graphs from edge lists, dense views, comparators."""
from __future__ import annotations

from contextlib import contextmanager

import numpy as np


@contextmanager
def tuned(handle, **knobs):
    """Set launch knobs of an fg Graph handle (fg_graph_tune) for the block,
    restoring the previous values afterwards."""
    old = {k: handle.get_tune(k) for k in knobs}
    for k, v in knobs.items():
        handle.tune(k, v)
    try:
        yield handle
    finally:
        for k, v in old.items():
            handle.tune(k, v)


def csr_from_edges(n_dst: int, edges, n_src: int | None = None):
    """Destination-major CSR from (src, dst) pairs; rows sorted ascending."""
    n_src = n_dst if n_src is None else n_src
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    order = np.lexsort((e[:, 0], e[:, 1]))   # by dst, then src
    e = e[order]
    row_ptr = np.zeros(n_dst + 1, np.int64)
    np.add.at(row_ptr, e[:, 1] + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    return row_ptr, e[:, 0].astype(np.int32)


def dense_adjacency(row_ptr, col_idx, n_src: int, values=None) -> np.ndarray:
    """A[v, u] (fp64): 1 (or the edge value) iff edge u -> v."""
    n_dst = len(row_ptr) - 1
    A = np.zeros((n_dst, n_src), np.float64)
    rows = np.repeat(np.arange(n_dst), np.diff(row_ptr))
    A[rows, col_idx] = 1.0 if values is None else values
    return A


def edge_rows(row_ptr) -> np.ndarray:
    return np.repeat(np.arange(len(row_ptr) - 1), np.diff(row_ptr))


def check_close(gpu, ref, abssum, tol=1e-4, what=""):
    """|gpu - ref| <= tol * abssum; where abssum == 0, exact equality
    (BASELINE.json north_star tolerance; SURVEY §8(c) comparator)."""
    gpu = np.asarray(gpu, np.float64)
    err = np.abs(gpu - ref)
    bound = tol * abssum
    bad = err > bound
    if bad.any():
        i = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {int(bad.sum())} elements out of tolerance; first at {tuple(i)}: "
                             f"gpu={gpu[tuple(i)]!r} ref={ref[tuple(i)]!r} abssum={abssum[tuple(i)]!r}")
    return float((err / np.where(abssum > 0, abssum, 1)).max()) if err.size else 0.0
