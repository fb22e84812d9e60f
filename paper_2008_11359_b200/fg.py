"""Thin ctypes binding of libfg.so (include/fg.h): argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; this module
only turns torch CUDA tensors into device pointers + sizes + the current CUDA
stream, and raises on a non-OK status.  There is no fallback: if libfg.so is
missing or CUDA is unavailable, calls fail loudly.

Names follow include/fg.h and the paper (§3.2): graph_create
(featgraph.spmat), spmm (featgraph.spmm), sddmm
(featgraph.sddmm), edge_softmax (GAT normalisation).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# FG_LIBFG: a development variant of libfg.so (tools/variants.py) -- same ABI
LIB_PATH = os.environ.get("FG_LIBFG") or os.path.join(_PKG, "lib", "libfg.so")

FG_OK, FG_EINVAL, FG_ESHAPE, FG_EUNSUPPORTED, FG_EGRAPH, FG_ECUDA, FG_ENOMEM, FG_ENCCL = range(8)
MSG = {"copy_u": 0, "u_mul_e": 1, "mlp": 2, "u_add_e": 3, "copy_e": 4}
REDUCE = {"sum": 0, "max": 1, "min": 2, "mean": 3}
EDGE = {"u_dot_v": 0, "u_add_v": 1, "u_sub_v": 2, "u_mul_v": 3}

# exported symbols declared in include/fg.h (checked by tests/test_abi.py)
SYMBOLS = ["fg_graph_create", "fg_graph_destroy", "fg_graph_info", "fg_graph_prepare", "fg_graph_prepare_hybrid",
           "fg_graph_hybrid_info", "fg_graph_tune",
           "fg_graph_get_tune", "fg_spmm_workspace_size", "fg_spmm",
           "fg_sddmm", "fg_edge_softmax", "fg_gat_attention", "fg_graph_transpose", "fg_spmm_backward", "fg_sddmm_backward",
           "fg_edge_softmax_backward", "fg_comm_unique_id", "fg_comm_init", "fg_comm_destroy",
           "fg_comm_info", "fg_allgather_rows", "fg_spmm_x16", "fg_sddmm_x16", "fg_sddmm_emul", "fg_dist_spmm", "fg_dist_sddmm", "fg_status_string", "fg_last_error", "fg_abi_version"]


# fg_tune_key (include/fg.h)
TUNE = {"l2_tile_mb": 0, "spmm_heavy_deg": 1, "balance_nnz": 2, "sddmm_seg_mb": 3, "sddmm_seg_min_mb": 4,
        "sddmm_persist": 5, "sddmm_l2_tile": 6, "sddmm_dot": 7, "gat_heavy_deg": 8, "mlp_impl": 9, "hybrid": 10,
        "spmm_seg_mb": 11, "sddmm_pipe": 12,
        "sddmm_order": 13, "sddmm_rb_mb": 14, "spmm_ldg256": 15}


class FGError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class GraphInfo(ctypes.Structure):
    _fields_ = [("n_dst", ctypes.c_int64), ("n_src", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("max_degree", ctypes.c_int64), ("n_empty_rows", ctypes.c_int64),
                ("n_sddmm_units", ctypes.c_int64), ("device_bytes", ctypes.c_int64)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libfg.so (raises if it was not built -- no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FGError(FG_ECUDA, f"libfg.so not built at {LIB_PATH}: run `python -m paper_2008_11359_b200.build`")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
    L.fg_graph_create.argtypes = [i64, i64, i64, vp, vp, vp, i32, vp, ctypes.POINTER(vp)]
    L.fg_graph_destroy.argtypes = [vp]
    L.fg_graph_info.argtypes = [vp, ctypes.POINTER(GraphInfo)]
    L.fg_graph_prepare.argtypes = [vp, i64, vp]
    L.fg_graph_prepare_hybrid.argtypes = [vp, i64, i64, vp]
    L.fg_graph_hybrid_info.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(ctypes.c_double)]
    L.fg_graph_tune.argtypes = [vp, i32, i64]
    L.fg_graph_get_tune.argtypes = [vp, i32, ctypes.POINTER(i64)]
    L.fg_spmm_workspace_size.argtypes = [vp, i32, i32, i32, i32, i32, ctypes.POINTER(sz)]
    L.fg_spmm.argtypes = [vp, i32, i32, i32, i32, vp, vp, vp, i32, vp, vp, vp, vp, vp, sz, vp]
    L.fg_sddmm.argtypes = [vp, i32, i32, i32, vp, vp, vp, vp]
    L.fg_spmm_x16.argtypes = [vp, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp]
    L.fg_sddmm_x16.argtypes = [vp, i32, i32, i32, vp, vp, vp, vp]
    L.fg_sddmm_emul.argtypes = [vp, i32, i32, vp, vp, vp, vp, vp]
    L.fg_dist_spmm.argtypes = [vp, vp, vp, i32, i32, i32, i32, vp, vp, vp, vp, i32, vp, vp, vp, vp, vp, sz, vp]
    L.fg_dist_sddmm.argtypes = [vp, vp, vp, i32, i32, i32, vp, vp, vp, vp, vp]
    L.fg_edge_softmax.argtypes = [vp, i32, vp, vp, vp]
    L.fg_gat_attention.argtypes = [vp, i32, i32, vp, vp, vp, vp, vp]
    L.fg_graph_transpose.argtypes = [vp, vp, ctypes.POINTER(vp)]
    L.fg_spmm_backward.argtypes = [vp, vp, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp]
    L.fg_sddmm_backward.argtypes = [vp, vp, i32, i32, i32, vp, vp, vp, vp, vp, vp]
    L.fg_edge_softmax_backward.argtypes = [vp, i32, vp, vp, vp, vp]
    L.fg_comm_unique_id.argtypes = [vp]
    L.fg_comm_init.argtypes = [vp, i32, i32, ctypes.POINTER(vp)]
    L.fg_comm_destroy.argtypes = [vp]
    L.fg_comm_info.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(i32)]
    L.fg_allgather_rows.argtypes = [vp, vp, i64, vp, vp, vp]
    for f in ["fg_graph_create", "fg_graph_destroy", "fg_graph_info", "fg_graph_prepare", "fg_graph_prepare_hybrid",
              "fg_graph_hybrid_info", "fg_graph_tune",
              "fg_graph_get_tune", "fg_spmm_workspace_size", "fg_spmm",
              "fg_sddmm", "fg_edge_softmax", "fg_gat_attention", "fg_graph_transpose", "fg_spmm_backward", "fg_sddmm_backward",
              "fg_edge_softmax_backward", "fg_comm_unique_id", "fg_comm_init", "fg_comm_destroy",
              "fg_comm_info", "fg_allgather_rows", "fg_spmm_x16", "fg_sddmm_x16", "fg_sddmm_emul", "fg_dist_spmm",
              "fg_dist_sddmm"]:
        getattr(L, f).restype = i32
    L.fg_status_string.argtypes = [i32]
    L.fg_status_string.restype = ctypes.c_char_p
    L.fg_last_error.restype = ctypes.c_char_p
    L.fg_abi_version.restype = i32
    _lib = L
    return L


def _check(status: int, what: str):
    if status != FG_OK:
        L = lib()
        raise FGError(status, f"{what}: {L.fg_status_string(status).decode()} -- {L.fg_last_error().decode()}")


def _ptr(t):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _dev(t, dtype, name):
    if t is None:
        return None
    if not t.is_cuda:
        raise FGError(FG_EINVAL, f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise FGError(FG_EINVAL, f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise FGError(FG_EINVAL, f"{name} must be contiguous")
    return t


def _head_dim(F: int, H: int) -> int:
    """D = F / H; F must split into H heads exactly (else the library would read
    rows with the wrong stride)."""
    if H < 1 or F % H != 0:
        raise FGError(FG_ESHAPE, f"feature width {F} does not split into H={H} heads")
    return F // H


def _out(t, shape, dtype, name):
    """A caller-supplied output tensor: CUDA, dtype, contiguous and exactly `shape`."""
    if t is None:
        return None
    t = _dev(t, dtype, name)
    if tuple(t.shape) != tuple(shape) and not (t.numel() == int(np.prod(shape)) and t.dim() == 1):
        raise FGError(FG_ESHAPE, f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    return t


class Graph:
    """fg_graph handle (featgraph.spmat).  Borrows row_ptr/col_idx/eid: the
    tensors are kept referenced by this object."""

    def __init__(self, row_ptr: torch.Tensor, col_idx: torch.Tensor, n_src: int | None = None,
                 eid: torch.Tensor | None = None, validate: bool = True, stream=None):
        self.row_ptr = _dev(row_ptr, torch.int64, "row_ptr")
        self.col_idx = _dev(col_idx, torch.int32, "col_idx")
        self.eid = _dev(eid, torch.int32, "eid")
        self.n_dst = row_ptr.numel() - 1
        self.n_src = self.n_dst if n_src is None else int(n_src)
        self.nnz = col_idx.numel()
        h = ctypes.c_void_p()
        _check(lib().fg_graph_create(self.n_dst, self.n_src, self.nnz, _ptr(self.row_ptr),
                                     _ptr(self.col_idx) if self.nnz else None, _ptr(self.eid),
                                     int(bool(validate)), _stream(stream), ctypes.byref(h)),
               "fg_graph_create")
        self.handle = h

    @classmethod
    def _from_handle(cls, h, n_dst, n_src, nnz):
        obj = cls.__new__(cls)
        obj.row_ptr = obj.col_idx = obj.eid = None   # owned by the library
        obj.n_dst, obj.n_src, obj.nnz, obj.handle = n_dst, n_src, nnz, h
        return obj

    def transpose(self, stream=None) -> "Graph":
        """fg_graph_transpose: the CSC handle (rows = sources) sharing edge ids."""
        h = ctypes.c_void_p()
        _check(lib().fg_graph_transpose(self.handle, _stream(stream), ctypes.byref(h)), "fg_graph_transpose")
        return Graph._from_handle(h, self.n_src, self.n_dst, self.nnz)

    def prepare(self, row_bytes: int, stream=None) -> "Graph":
        """fg_graph_prepare: build the source-segment tables of the gSDDMM traversal
        and of the segmented u_mul_e-sum passes for gathered rows of `row_bytes`
        bytes (synchronous; no-op when that width is not segmented).  Call before
        timing / CUDA-graph capture."""
        _check(lib().fg_graph_prepare(self.handle, int(row_bytes), _stream(stream)), "fg_graph_prepare")
        return self

    def prepare_hybrid(self, row_bytes: int, smem_bytes: int = 48 * 1024, stream=None) -> "Graph":
        """fg_graph_prepare_hybrid: stage the smem_bytes // row_bytes sources of
        highest out-degree in shared memory for copy_u-sum; enable
        with tune("hybrid", 1).  Synchronous."""
        _check(lib().fg_graph_prepare_hybrid(self.handle, int(row_bytes), int(smem_bytes), _stream(stream)),
               "fg_graph_prepare_hybrid")
        return self

    def hybrid_info(self) -> tuple[int, float]:
        k, share = ctypes.c_int64(0), ctypes.c_double(0)
        _check(lib().fg_graph_hybrid_info(self.handle, ctypes.byref(k), ctypes.byref(share)), "fg_graph_hybrid_info")
        return int(k.value), float(share.value)

    def tune(self, key: str, value: int) -> "Graph":
        """fg_graph_tune: set one launch knob of this handle (include/fg.h fg_tune_key)."""
        _check(lib().fg_graph_tune(self.handle, TUNE[key], int(value)), f"fg_graph_tune({key})")
        return self

    def get_tune(self, key: str) -> int:
        v = ctypes.c_int64(0)
        _check(lib().fg_graph_get_tune(self.handle, TUNE[key], ctypes.byref(v)), f"fg_graph_get_tune({key})")
        return int(v.value)

    def info(self) -> GraphInfo:
        inf = GraphInfo()
        _check(lib().fg_graph_info(self.handle, ctypes.byref(inf)), "fg_graph_info")
        return inf

    def close(self):
        if getattr(self, "handle", None):
            lib().fg_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def spmm(g: Graph, msg: str, reduce: str, X: torch.Tensor, *, H: int = 1, E: torch.Tensor | None = None,
         W: torch.Tensor | None = None, X_dst: torch.Tensor | None = None, out: torch.Tensor | None = None,
         arg_u: torch.Tensor | bool | None = None, arg_e: torch.Tensor | bool | None = None, stream=None):
    """featgraph.spmm (Eq. (1)).  Returns out, or (out, arg_u, arg_e) when args requested.
    copy_e takes X=None and E [nnz][F].  A torch.bfloat16 X selects bf16 feature
    storage (fg_spmm_x16: copy_u / u_mul_e, any reducer; fp32 arithmetic and out)."""
    if X is not None and X.dtype == torch.bfloat16:
        return _spmm_x16(g, msg, reduce, X, H=H, E=E, out=out, arg_u=arg_u, arg_e=arg_e, stream=stream)
    X = _dev(X, torch.float32, "X")
    E, W, X_dst = _dev(E, torch.float32, "E"), _dev(W, torch.float32, "W"), _dev(X_dst, torch.float32, "X_dst")
    if msg == "copy_e":
        d_in = 0
        F = E.numel() // max(E.shape[0], 1) if E.dim() > 1 else 1
        H_, D = H, _head_dim(F, H)
    elif msg == "mlp":
        d_in, F = W.shape
        H_, D = 1, F
    else:
        d_in = 0
        F = X.numel() // max(X.shape[0], 1) if X.dim() > 1 else 1
        H_, D = H, _head_dim(F, H)
    if X is not None and msg != "copy_e" and X.shape[0] < g.n_src:
        raise FGError(FG_ESHAPE, f"X has {X.shape[0]} rows, the graph has {g.n_src} sources")
    if msg == "mlp":
        if X.numel() != X.shape[0] * d_in or (X_dst is not None and X_dst.numel() != g.n_dst * d_in):
            raise FGError(FG_ESHAPE, f"mlp: X / X_dst rows must have d_in={d_in} features")
    elif msg in ("u_mul_e", "u_add_e") and E is not None and E.numel() != g.nnz * H_:
        raise FGError(FG_ESHAPE, f"E has {E.numel()} elements, expected nnz*H = {g.nnz * H_}")
    elif msg == "copy_e" and E is not None and E.shape[0] != g.nnz:
        raise FGError(FG_ESHAPE, f"E has {E.shape[0]} rows, expected nnz = {g.nnz}")
    device = (X if X is not None else E).device
    out = _out(out, (g.n_dst, F), torch.float32, "out")
    if out is None:
        out = torch.empty((g.n_dst, F), dtype=torch.float32, device=device)
    want = reduce in ("max", "min") and (arg_u is not None or arg_e is not None)
    if arg_u is True:
        arg_u = torch.empty((g.n_dst, F), dtype=torch.int32, device=device)
    if arg_e is True:
        arg_e = torch.empty((g.n_dst, F), dtype=torch.int32, device=device)
    arg_u = _out(arg_u, (g.n_dst, F), torch.int32, "arg_u") if isinstance(arg_u, torch.Tensor) else None
    arg_e = _out(arg_e, (g.n_dst, F), torch.int32, "arg_e") if isinstance(arg_e, torch.Tensor) else None
    _check(lib().fg_spmm(g.handle, MSG[msg], REDUCE[reduce], H_, D, _ptr(X), _ptr(E), _ptr(W), d_in, _ptr(X_dst),
                         _ptr(out), _ptr(arg_u), _ptr(arg_e), None, 0, _stream(stream)),
           f"fg_spmm({msg},{reduce})")
    if want:
        return out, arg_u, arg_e
    return out


def _spmm_x16(g, msg, reduce, X, *, H, E, out, arg_u, arg_e, stream):
    X = _dev(X, torch.bfloat16, "X")
    E = _dev(E, torch.float32, "E")
    F = X.numel() // max(X.shape[0], 1) if X.dim() > 1 else 1
    out = _out(out, (g.n_dst, F), torch.float32, "out")
    if out is None:
        out = torch.empty((g.n_dst, F), dtype=torch.float32, device=X.device)
    want = reduce in ("max", "min") and (arg_u is not None or arg_e is not None)
    if arg_u is True:
        arg_u = torch.empty((g.n_dst, F), dtype=torch.int32, device=X.device)
    if arg_e is True:
        arg_e = torch.empty((g.n_dst, F), dtype=torch.int32, device=X.device)
    arg_u = _out(arg_u, (g.n_dst, F), torch.int32, "arg_u") if isinstance(arg_u, torch.Tensor) else None
    arg_e = _out(arg_e, (g.n_dst, F), torch.int32, "arg_e") if isinstance(arg_e, torch.Tensor) else None
    _check(lib().fg_spmm_x16(g.handle, MSG[msg], REDUCE[reduce], H, _head_dim(F, H), _ptr(X), _ptr(E), _ptr(out),
                             _ptr(arg_u), _ptr(arg_e), _stream(stream)), f"fg_spmm_x16({msg},{reduce})")
    return (out, arg_u, arg_e) if want else out


def sddmm(g: Graph, X: torch.Tensor, Y: torch.Tensor | None = None, *, H: int = 1, op: str = "u_dot_v",
          out: torch.Tensor | None = None, E: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """featgraph.sddmm (Eq. (4), Fig. 5): out[eid][h] = <X[u,h,:], Y[v,h,:]> for
    op="u_dot_v"; the elementwise ops u_add_v / u_sub_v / u_mul_v give
    out[eid][j] = X[u][j] OP Y[v][j] ([nnz][F]).  torch.bfloat16 X (and Y)
    select bf16 feature storage (fg_sddmm_x16, u_dot_v; fp32 arithmetic and out).
    E [nnz][H] (op="u_dot_v", fp32 X): u_dot_v-then-e_mul, out = score * E
    (fg_sddmm_emul)."""
    if E is not None:
        if op != "u_dot_v":
            raise FGError(FG_EINVAL, "sddmm: E (e_mul) applies to u_dot_v only")
        X = _dev(X, torch.float32, "X")
        Y = X if Y is None else _dev(Y, torch.float32, "Y")
        E = _dev(E, torch.float32, "E")
        F = X.numel() // max(X.shape[0], 1)
        E = _out(E, (g.nnz, H), torch.float32, "E")
        out = _out(out, (g.nnz, H), torch.float32, "out")
        if out is None:
            out = torch.empty((g.nnz, H), dtype=torch.float32, device=X.device)
        _check(lib().fg_sddmm_emul(g.handle, H, _head_dim(F, H), _ptr(X), _ptr(Y), _ptr(E), _ptr(out), _stream(stream)),
               "fg_sddmm_emul")
        return out
    if X.dtype == torch.bfloat16:
        X = _dev(X, torch.bfloat16, "X")
        Y = X if Y is None else _dev(Y, torch.bfloat16, "Y")
        F = X.numel() // max(X.shape[0], 1)
        out = _out(out, (g.nnz, H), torch.float32, "out")
        if out is None:
            out = torch.empty((g.nnz, H), dtype=torch.float32, device=X.device)
        _check(lib().fg_sddmm_x16(g.handle, EDGE[op], H, _head_dim(F, H), _ptr(X), _ptr(Y), _ptr(out), _stream(stream)),
               "fg_sddmm_x16")
        return out
    X = _dev(X, torch.float32, "X")
    Y = X if Y is None else _dev(Y, torch.float32, "Y")
    F = X.numel() // max(X.shape[0], 1)
    oshape = (g.nnz, H if op == "u_dot_v" else F)
    out = _out(out, oshape, torch.float32, "out")
    if out is None:
        out = torch.empty(oshape, dtype=torch.float32, device=X.device)
    _check(lib().fg_sddmm(g.handle, EDGE[op], H, _head_dim(F, H), _ptr(X), _ptr(Y), _ptr(out), _stream(stream)), "fg_sddmm")
    return out


def edge_softmax(g: Graph, scores: torch.Tensor, *, H: int = 1, out: torch.Tensor | None = None,
                 stream=None) -> torch.Tensor:
    """Per-destination softmax over in-edges, per head (GAT)."""
    scores = _out(scores, (g.nnz, H), torch.float32, "scores")
    out = _out(out, (g.nnz, H), torch.float32, "out")
    if out is None:
        out = torch.empty_like(scores)
    _check(lib().fg_edge_softmax(g.handle, H, _ptr(scores), _ptr(out), _stream(stream)), "fg_edge_softmax")
    return out


def gat_attention(g: Graph, X: torch.Tensor, Y: torch.Tensor | None = None, *, H: int = 1,
                  out: torch.Tensor | None = None, scores: torch.Tensor | bool | None = None, stream=None):
    """Fused GAT layer: u_dot_v -> edge softmax -> u_mul_e-sum in one pass.
    Returns out (and the pre-softmax scores when scores=True or a tensor)."""
    X = _dev(X, torch.float32, "X")
    Y = X if Y is None else _dev(Y, torch.float32, "Y")
    F = X.shape[1]
    out = _out(out, (g.n_dst, F), torch.float32, "out")
    if out is None:
        out = torch.empty((g.n_dst, F), dtype=torch.float32, device=X.device)
    want = scores is not None and scores is not False
    if scores is True:
        scores = torch.empty((g.nnz, H), dtype=torch.float32, device=X.device)
    sc = _out(scores, (g.nnz, H), torch.float32, "scores") if isinstance(scores, torch.Tensor) else None
    _check(lib().fg_gat_attention(g.handle, H, _head_dim(F, H), _ptr(X), _ptr(Y), _ptr(out), _ptr(sc), _stream(stream)),
           "fg_gat_attention")
    return (out, sc) if want else out


# ------------------------------------------------------------------ backward
def spmm_backward(g: Graph, gT: Graph | None, msg: str, reduce: str, dOut: torch.Tensor, *, H: int = 1,
                  X: torch.Tensor | None = None, E: torch.Tensor | None = None, arg_u: torch.Tensor | None = None,
                  want_dX: bool = True, want_dE: bool = False, stream=None):
    """Gradients of fg_spmm (copy_u / u_mul_e).  Returns (dX, dE)."""
    dOut = _dev(dOut, torch.float32, "dOut")
    F = dOut.shape[1]
    dX = torch.empty((g.n_src, F), dtype=torch.float32, device=dOut.device) if want_dX else None
    dE = torch.empty((g.nnz, H), dtype=torch.float32, device=dOut.device) if want_dE else None
    _check(lib().fg_spmm_backward(g.handle, gT.handle if gT is not None else None, MSG[msg], REDUCE[reduce], H,
                                  _head_dim(F, H), _ptr(_dev(X, torch.float32, "X")), _ptr(_dev(E, torch.float32, "E")),
                                  _ptr(dOut), _ptr(_dev(arg_u, torch.int32, "arg_u")), _ptr(dX), _ptr(dE),
                                  _stream(stream)), "fg_spmm_backward")
    return dX, dE


def sddmm_backward(g: Graph, gT: Graph | None, X: torch.Tensor, Y: torch.Tensor, dS: torch.Tensor, *, H: int = 1,
                   want_dX: bool = True, want_dY: bool = True, stream=None):
    """Gradients of fg_sddmm(u_dot_v) w.r.t. X (sources) and Y (destinations)."""
    X, Y, dS = _dev(X, torch.float32, "X"), _dev(Y, torch.float32, "Y"), _dev(dS, torch.float32, "dS")
    F = X.shape[1]
    dX = torch.empty((g.n_src, F), dtype=torch.float32, device=X.device) if want_dX else None
    dY = torch.empty((g.n_dst, F), dtype=torch.float32, device=X.device) if want_dY else None
    _check(lib().fg_sddmm_backward(g.handle, gT.handle if gT is not None else None, EDGE["u_dot_v"], H, _head_dim(F, H),
                                   _ptr(X), _ptr(Y), _ptr(dS), _ptr(dX), _ptr(dY), _stream(stream)),
           "fg_sddmm_backward")
    return dX, dY


def edge_softmax_backward(g: Graph, alpha: torch.Tensor, dalpha: torch.Tensor, *, H: int = 1, stream=None):
    alpha, dalpha = _dev(alpha, torch.float32, "alpha"), _dev(dalpha, torch.float32, "dalpha")
    ds = torch.empty_like(alpha)
    _check(lib().fg_edge_softmax_backward(g.handle, H, _ptr(alpha), _ptr(dalpha), _ptr(ds), _stream(stream)),
           "fg_edge_softmax_backward")
    return ds


# ------------------------------------------------------------------ multi-GPU
def comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().fg_comm_unique_id(buf), "fg_comm_unique_id")
    return buf.raw


class Comm:
    def __init__(self, unique_id: bytes, nranks: int, rank: int):
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(unique_id, 128)
        _check(lib().fg_comm_init(buf, nranks, rank, ctypes.byref(h)), "fg_comm_init")
        self.handle, self.nranks, self.rank = h, nranks, rank

    def nranks_nccl(self) -> int:
        """The communicator size as NCCL reports it (fg_comm_info)."""
        n, r = ctypes.c_int(0), ctypes.c_int(0)
        _check(lib().fg_comm_info(self.handle, ctypes.byref(n), ctypes.byref(r)), "fg_comm_info")
        return int(n.value)

    def allgather_rows(self, shard_offsets, X_local: torch.Tensor | None, X_full: torch.Tensor, stream=None):
        import numpy as np
        off = np.ascontiguousarray(np.asarray(shard_offsets, dtype=np.int64))
        row_elems = X_full.numel() // max(X_full.shape[0], 1)
        _check(lib().fg_allgather_rows(self.handle, ctypes.c_void_p(off.ctypes.data), row_elems, _ptr(X_local),
                                       _ptr(X_full), _stream(stream)), "fg_allgather_rows")
        return X_full

    def dist_spmm(self, g_local: "Graph", shard_offsets, msg: str, reduce: str, X_local: torch.Tensor,
                  X_full: torch.Tensor, *, H: int = 1, E: torch.Tensor | None = None, out: torch.Tensor | None = None,
                  stream=None) -> torch.Tensor:
        """fg_dist_spmm (sum / mean reducers of copy_u / u_mul_e / u_add_e): all-gather
        X_local into X_full, then the local gSpMM on this rank's rows."""
        import numpy as np
        off = np.ascontiguousarray(np.asarray(shard_offsets, dtype=np.int64))
        X_full = _dev(X_full, torch.float32, "X_full")
        E = _dev(E, torch.float32, "E")
        F = X_full.numel() // max(X_full.shape[0], 1)
        if out is None:
            out = torch.empty((g_local.n_dst, F), dtype=torch.float32, device=X_full.device)
        _check(lib().fg_dist_spmm(g_local.handle, self.handle, ctypes.c_void_p(off.ctypes.data), MSG[msg],
                                  REDUCE[reduce], H, _head_dim(F, H), _ptr(X_local), _ptr(X_full), _ptr(E), None, 0, None,
                                  _ptr(out), None, None, None, 0, _stream(stream)), "fg_dist_spmm")
        return out

    def dist_sddmm(self, g_local: "Graph", shard_offsets, X_local: torch.Tensor, X_full: torch.Tensor,
                   Y_local: torch.Tensor, *, H: int = 1, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """fg_dist_sddmm (u_dot_v): all-gather X_local into X_full, then the local gSDDMM."""
        import numpy as np
        off = np.ascontiguousarray(np.asarray(shard_offsets, dtype=np.int64))
        X_full = _dev(X_full, torch.float32, "X_full")
        Y_local = _dev(Y_local, torch.float32, "Y_local")
        F = X_full.numel() // max(X_full.shape[0], 1)
        if out is None:
            out = torch.empty((g_local.nnz, H), dtype=torch.float32, device=X_full.device)
        _check(lib().fg_dist_sddmm(g_local.handle, self.handle, ctypes.c_void_p(off.ctypes.data), EDGE["u_dot_v"], H,
                                   _head_dim(F, H), _ptr(X_local), _ptr(X_full), _ptr(Y_local), _ptr(out), _stream(stream)),
               "fg_dist_sddmm")
        return out

    def close(self):
        if self.handle:
            lib().fg_comm_destroy(self.handle)
            self.handle = None
