"""fp64 CPU oracle for the FeatGraph hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  It shares no code with the
CUDA path (paper_2008_11359_b200/); see oracle/oracle.c for the definitions and
the PAPER.md passages each routine follows.  Pins: tests/test_oracle_pins.py.

Parity status per function:
  spmm copy_u sum/max, u_mul_e sum/max, mlp max/sum, sddmm u_dot_v,
  sddmm u_dot_v-then-e_mul, edge_softmax -- all pinned (no "parity unpinned"
  functions).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

OPS = {"copy_u": 0, "u_mul_e": 1, "mlp": 2, "u_add_e": 3, "copy_e": 4}
REDS = {"sum": 0, "max": 1, "min": 2, "mean": 3}


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-Wall",
                               "-o", _SO, src, "-lm"])
    return _SO


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64, i32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        lib.or_spmm.argtypes = [i64, vp, vp, vp, vp, i32, i32, i32, i32, vp, vp, vp, i32, vp,
                                vp, vp, vp, vp]
        lib.or_spmm.restype = None
        lib.or_sddmm.argtypes = [i64, vp, vp, vp, i32, i32, vp, vp, vp, vp]
        lib.or_sddmm.restype = None
        lib.or_edge_softmax.argtypes = [i64, vp, vp, vp, i32, vp, vp]
        lib.or_edge_softmax.restype = None
        lib.or_sddmm_binary.argtypes = [i64, vp, vp, vp, i32, i64, vp, vp, vp, vp]
        lib.or_sddmm_binary.restype = None
        lib.or_sddmm_emul.argtypes = [i64, vp, vp, vp, vp, i32, i32, vp, vp, vp, vp, vp]
        lib.or_sddmm_emul.restype = None
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _c(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt)


def _rows(rows, n_dst):
    if rows is None:
        return n_dst, None
    rows = _c(rows, np.int64)
    return rows.size, rows


def spmm(row_ptr, col_idx, op: str, red: str, X, *, H: int = 1, D: int | None = None, E=None,
         W=None, X_dst=None, eid=None, rows=None, want_arg: bool = True):
    """Eq. (1) for the listed destination rows.  Returns (ref, abssum, arg_u, arg_e)
    with ref/abssum fp64 [n_rows][F] and args int32 (max/min only, else None)."""
    row_ptr, col_idx, eid = _c(row_ptr, np.int64), _c(col_idx, np.int32), _c(eid, np.int32)
    X = _c(X, np.float32)
    n_dst = row_ptr.size - 1
    d_in = 0
    if op == "copy_e":                      # message = the edge's own feature row
        E = _c(E, np.float32)
        F = E.reshape(E.shape[0], -1).shape[1]
        D = F // H if D is None else D
        assert H * D == F
    elif op == "mlp":
        W = _c(W, np.float32)
        d_in, F = W.shape
        H, D = 1, F
        X_dst = X if X_dst is None else _c(X_dst, np.float32)
        X = X.reshape(-1, d_in)
    else:
        F = X.reshape(X.shape[0], -1).shape[1]
        D = F // H if D is None else D
        assert H * D == F
    E = _c(E, np.float32)
    n_rows, rows_a = _rows(rows, n_dst)
    ref = np.empty((n_rows, F), np.float64)
    ab = np.empty((n_rows, F), np.float64)
    au = ae = None
    if red in ("max", "min") and want_arg:
        au = np.empty((n_rows, F), np.int32)
        ae = np.empty((n_rows, F), np.int32)
    _L().or_spmm(n_rows, _p(rows_a), _p(row_ptr), _p(col_idx), _p(eid), OPS[op], REDS[red], H, D,
                 _p(X), _p(E), _p(W), d_in, _p(X_dst), _p(ref), _p(ab), _p(au), _p(ae))
    return ref, ab, au, ae


def sddmm(row_ptr, col_idx, X, Y=None, *, H: int = 1, rows=None):
    """Eq. (4) / Fig. 5 u_dot_v for the edges of the listed rows, in CSR order of
    the listed rows.  Returns (ref, abssum) fp64 [edges][H]."""
    row_ptr, col_idx = _c(row_ptr, np.int64), _c(col_idx, np.int32)
    X = _c(X, np.float32)
    Y = X if Y is None else _c(Y, np.float32)
    F = X.reshape(X.shape[0], -1).shape[1]
    D = F // H
    n_rows, rows_a = _rows(rows, row_ptr.size - 1)
    ne = int((row_ptr[1:] - row_ptr[:-1]).sum()) if rows_a is None else \
        int((row_ptr[rows_a + 1] - row_ptr[rows_a]).sum())
    ref = np.empty((ne, H), np.float64)
    ab = np.empty((ne, H), np.float64)
    _L().or_sddmm(n_rows, _p(rows_a), _p(row_ptr), _p(col_idx), H, D, _p(X), _p(Y), _p(ref), _p(ab))
    return ref, ab


def sddmm_emul(row_ptr, col_idx, X, Y, E, *, H: int = 1, eid=None, rows=None):
    """u_dot_v then e_mul (oracle.c or_sddmm_emul): (Eq. (4) score) * E[eid][h]
    for the edges of the listed rows, in CSR order of the listed rows.  Returns
    (ref, abssum) fp64 [edges][H]."""
    row_ptr, col_idx = _c(row_ptr, np.int64), _c(col_idx, np.int32)
    X = _c(X, np.float32)
    Y = X if Y is None else _c(Y, np.float32)
    E = _c(E, np.float32)
    eid = _c(eid, np.int32)
    F = X.reshape(X.shape[0], -1).shape[1]
    D = F // H
    n_rows, rows_a = _rows(rows, row_ptr.size - 1)
    ne = int((row_ptr[1:] - row_ptr[:-1]).sum()) if rows_a is None else \
        int((row_ptr[rows_a + 1] - row_ptr[rows_a]).sum())
    ref = np.empty((ne, H), np.float64)
    ab = np.empty((ne, H), np.float64)
    _L().or_sddmm_emul(n_rows, _p(rows_a), _p(row_ptr), _p(col_idx), _p(eid), H, D, _p(X), _p(Y), _p(E),
                       _p(ref), _p(ab))
    return ref, ab


BINOPS = {"u_add_v": 0, "u_sub_v": 1, "u_mul_v": 2}


def sddmm_binary(row_ptr, col_idx, op: str, X, Y=None, *, rows=None):
    """Elementwise SDDMM X[u] OP Y[v] (OP in add/sub/mul) for the edges of the
    listed rows in CSR order.  Returns (ref, abssum) fp64 [edges][F]."""
    row_ptr, col_idx = _c(row_ptr, np.int64), _c(col_idx, np.int32)
    X = _c(X, np.float32)
    Y = X if Y is None else _c(Y, np.float32)
    F = X.reshape(X.shape[0], -1).shape[1]
    n_rows, rows_a = _rows(rows, row_ptr.size - 1)
    ne = int(row_ptr[-1] - row_ptr[0]) if rows_a is None else \
        int((row_ptr[rows_a + 1] - row_ptr[rows_a]).sum())
    ref = np.empty((ne, F), np.float64)
    ab = np.empty((ne, F), np.float64)
    _L().or_sddmm_binary(n_rows, _p(rows_a), _p(row_ptr), _p(col_idx), BINOPS[op], F, _p(X), _p(Y), _p(ref),
                         _p(ab))
    return ref, ab


def edge_softmax(row_ptr, scores, *, H: int = 1, eid=None, rows=None):
    """Per-destination, per-head softmax over in-edges.  scores fp32 [nnz][H]
    indexed by edge id.  Returns alpha fp64 [edges of listed rows][H] in CSR
    order of the listed rows."""
    row_ptr, eid = _c(row_ptr, np.int64), _c(eid, np.int32)
    S = _c(scores, np.float32)
    n_rows, rows_a = _rows(rows, row_ptr.size - 1)
    ne = int(row_ptr[-1] - row_ptr[0]) if rows_a is None else \
        int((row_ptr[rows_a + 1] - row_ptr[rows_a]).sum())
    alpha = np.empty((ne, H), np.float64)
    _L().or_edge_softmax(n_rows, _p(rows_a), _p(row_ptr), _p(eid), H, _p(S), _p(alpha))
    return alpha


def edge_positions(row_ptr, rows) -> np.ndarray:
    """CSR positions of the edges of `rows`, in the order the oracle emits them."""
    row_ptr = np.asarray(row_ptr, np.int64)
    rows = np.asarray(rows, np.int64)
    if rows.size == 0:
        return np.zeros(0, np.int64)
    starts, ends = row_ptr[rows], row_ptr[rows + 1]
    lens = ends - starts
    idx = np.repeat(starts - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens)
    return idx + np.arange(lens.sum())


# ------------------------------------------------------------------ backward (gradient duality)
def _bind_backward():
    lib = _L()
    if getattr(lib, "_bw_bound", False):
        return lib
    i64, i32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
    lib.or_spmm_backward.argtypes = [i64, i64, i64, vp, vp, vp, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp]
    lib.or_spmm_backward.restype = None
    lib.or_sddmm_backward.argtypes = [i64, i64, vp, vp, vp, i32, i32, vp, vp, vp, vp, vp]
    lib.or_sddmm_backward.restype = None
    lib.or_edge_softmax_backward.argtypes = [i64, vp, vp, i32, vp, vp, vp]
    lib.or_edge_softmax_backward.restype = None
    lib._bw_bound = True
    return lib


def spmm_backward(row_ptr, col_idx, op: str, red: str, X, dOut, *, n_src: int, H: int = 1, E=None, eid=None,
                  arg_u=None, want_dE: bool = False):
    """Gradients of Eq. (1) (copy_u / u_mul_e; sum / max / min / mean).  Returns (dX, dE) fp64."""
    row_ptr, col_idx, eid = _c(row_ptr, np.int64), _c(col_idx, np.int32), _c(eid, np.int32)
    X, dOut, E = _c(X, np.float32), _c(dOut, np.float32), _c(E, np.float32)
    arg_u = _c(arg_u, np.int32)
    n_dst = row_ptr.size - 1
    nnz = int(row_ptr[-1])
    F = dOut.reshape(n_dst, -1).shape[1] if n_dst else X.reshape(n_src, -1).shape[1]
    D = F // H
    dX = np.empty((n_src, F), np.float64)
    dE = np.empty((nnz, H), np.float64) if want_dE else None
    _bind_backward().or_spmm_backward(n_dst, n_src, nnz, _p(row_ptr), _p(col_idx), _p(eid), OPS[op], REDS[red], H,
                                      D, _p(X), _p(E), _p(dOut), _p(arg_u), _p(dX), _p(dE))
    return dX, dE


def sddmm_backward(row_ptr, col_idx, X, Y, dS, *, H: int = 1, eid=None):
    """Gradients of Eq. (4) u_dot_v w.r.t. X (sources) and Y (destinations), fp64."""
    row_ptr, col_idx, eid = _c(row_ptr, np.int64), _c(col_idx, np.int32), _c(eid, np.int32)
    X, Y, dS = _c(X, np.float32), _c(Y, np.float32), _c(dS, np.float32)
    n_dst, n_src = row_ptr.size - 1, X.shape[0]
    F = X.reshape(n_src, -1).shape[1]
    dX = np.empty((n_src, F), np.float64)
    dY = np.empty((n_dst, F), np.float64)
    _bind_backward().or_sddmm_backward(n_dst, n_src, _p(row_ptr), _p(col_idx), _p(eid), H, F // H, _p(X), _p(Y),
                                       _p(dS), _p(dX), _p(dY))
    return dX, dY


def edge_softmax_backward(row_ptr, alpha, dalpha, *, H: int = 1, eid=None):
    row_ptr, eid = _c(row_ptr, np.int64), _c(eid, np.int32)
    alpha, dalpha = _c(alpha, np.float32), _c(dalpha, np.float32)
    ds = np.empty(alpha.shape, np.float64)
    _bind_backward().or_edge_softmax_backward(row_ptr.size - 1, _p(row_ptr), _p(eid), H, _p(alpha), _p(dalpha),
                                              _p(ds))
    return ds


def gat(row_ptr, col_idx, X, Y=None, *, H: int = 1):
    """Fused GAT layer definition (sddmm -> edge softmax -> u_mul_e-sum), fp64.
    Returns (ref, abssum) [n_dst][H*D]."""
    row_ptr, col_idx = _c(row_ptr, np.int64), _c(col_idx, np.int32)
    X = _c(X, np.float32)
    Y = X if Y is None else _c(Y, np.float32)
    n_dst = row_ptr.size - 1
    F = X.reshape(X.shape[0], -1).shape[1]
    lib = _L()
    if not getattr(lib, "_gat_bound", False):
        i64, i32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        lib.or_gat.argtypes = [i64, vp, vp, i32, i32, vp, vp, vp, vp]
        lib.or_gat.restype = None
        lib._gat_bound = True
    ref = np.empty((n_dst, F), np.float64)
    ab = np.empty((n_dst, F), np.float64)
    lib.or_gat(n_dst, _p(row_ptr), _p(col_idx), H, F // H, _p(X), _p(Y), _p(ref), _p(ab))
    return ref, ab
