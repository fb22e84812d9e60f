"""Seeded synthetic inputs (graphs + features) shared by tests, smoke() and bench.py.

This module holds NONE of the method's arithmetic -- only random numbers,
degree sequences and neighbour sampling (gen/gen.c).  Both the oracle tests and
the CUDA path draw their inputs from here; neither side's results feed back.

Recipe:
  * destination-major CSR (row v = in-neighbours of v, ascending), int64 row_ptr,
    int32 col_idx (Eq. (3));
  * in-degrees: lognormal rescaled to sum to m exactly (reddit / proteins shapes,
    SURVEY L11) or the rand-100K two-block rule;
  * sources: Chung-Lu (probability proportional to the source's own degree),
    drawn without replacement, or uniform (`uniform_sources`);
  * features: real regime U[-1,1) in multiples of 2^-23; integer regime small
    integers so every sum is exact in fp32.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libfggen.so")
_lib = None

SEED_BASE = 200811359  # graph seed = 200811359 + config index


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-Wall",
                               "-o", _SO, src, "-lm"])
    return _SO


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64, u64, i32, dbl, vp = (ctypes.c_int64, ctypes.c_uint64, ctypes.c_int,
                                  ctypes.c_double, ctypes.c_void_p)
        lib.fggen_features.argtypes = [i64, u64, u64, i32, i64, i64, dbl, vp]
        lib.fggen_features.restype = None
        lib.fggen_degrees_lognormal.argtypes = [i64, i64, dbl, i64, i64, u64, vp]
        lib.fggen_degrees_lognormal.restype = i32
        lib.fggen_degrees_two_block.argtypes = [i64, i64, i64, i64, u64, vp]
        lib.fggen_degrees_two_block.restype = None
        lib.fggen_permutation.argtypes = [i64, u64, u64, vp]
        lib.fggen_permutation.restype = None
        lib.fggen_fill_csr.argtypes = [i64, i64, vp, vp, u64, vp, vp]
        lib.fggen_fill_csr.restype = i32
        lib.fggen_rand_u64.argtypes = [u64, u64, u64]
        lib.fggen_rand_u64.restype = u64
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


# ------------------------------------------------------------------ features
REAL, UNIT, INT, SCALED = 0, 1, 2, 3


def features(shape, seed: int, stream: int, regime: int = REAL, lo: int = -8, hi: int = 8,
             scale: float = 1.0) -> np.ndarray:
    """fp32 array of `shape`.  REAL: U[-1,1) multiples of 2^-23; UNIT: U[0,1);
    INT: integers in [lo, hi]; SCALED: U[-scale, scale)."""
    out = np.empty(int(np.prod(shape)) if len(shape) else 1, dtype=np.float32)
    _L().fggen_features(out.size, seed, stream, regime, lo, hi, scale, _ptr(out))
    return out.reshape(shape)


# ------------------------------------------------------------------ graphs
@dataclass
class Graph:
    n_dst: int
    n_src: int
    row_ptr: np.ndarray  # int64 [n_dst+1]
    col_idx: np.ndarray  # int32 [nnz]
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def degrees(self) -> np.ndarray:
        return np.diff(self.row_ptr)


def degrees_lognormal(n: int, m: int, sigma: float, dmax: int, seed: int, dmin: int = 1) -> np.ndarray:
    deg = np.empty(max(n, 1), dtype=np.int64)[:n]
    rc = _L().fggen_degrees_lognormal(n, m, sigma, dmin, dmax, seed, _ptr(deg))
    if rc != 0:
        raise ValueError(f"lognormal degrees: m={m} unreachable for n={n}, d in [{dmin},{dmax}]")
    return deg


def degrees_two_block(n_high: int, deg_high: int, n_low: int, deg_low: int, seed: int) -> np.ndarray:
    deg = np.empty(n_high + n_low, dtype=np.int64)
    _L().fggen_degrees_two_block(n_high, deg_high, n_low, deg_low, seed, _ptr(deg))
    return deg


def permutation(n: int, seed: int, stream: int = 7) -> np.ndarray:
    p = np.empty(n, dtype=np.int64)
    _L().fggen_permutation(n, seed, stream, _ptr(p))
    return p


def csr_from_degrees(deg: np.ndarray, n_src: int, seed: int, uniform_sources: bool = False,
                     weights: np.ndarray | None = None, name: str = "") -> Graph:
    deg = np.ascontiguousarray(deg, dtype=np.int64)
    n_dst = deg.size
    row_ptr = np.zeros(n_dst + 1, dtype=np.int64)
    np.cumsum(deg, out=row_ptr[1:])
    col_idx = np.empty(max(int(row_ptr[-1]), 1), dtype=np.int32)
    if uniform_sources:
        w = None
    else:
        if weights is None:
            # Chung-Lu: weight of source u = its own target degree (square graphs)
            if n_src != n_dst:
                raise ValueError("Chung-Lu weights need n_src == n_dst; pass weights")
            weights = deg
        w = np.ascontiguousarray(weights, dtype=np.float64)
        if w.sum() <= 0:
            w = None
    rc = _L().fggen_fill_csr(n_dst, n_src, _ptr(deg), _ptr(w) if w is not None else None, seed,
                             _ptr(row_ptr), _ptr(col_idx))
    if rc != 0:
        raise ValueError("a degree exceeds the number of sources")
    return Graph(n_dst, n_src, row_ptr, col_idx[: int(row_ptr[-1])], name)


def random_graph(n: int, m: int, seed: int, sigma: float = 1.0, dmax: int | None = None,
                 uniform_sources: bool = False, n_empty: int = 0, name: str = "random") -> Graph:
    """Small lognormal graph for tests; `n_empty` rows (seeded positions) get degree 0."""
    dmax = n if dmax is None else dmax
    deg = np.zeros(n, np.int64)
    keep = np.sort(permutation(n, seed, 11)[: n - n_empty])
    deg[keep] = degrees_lognormal(n - n_empty, m, sigma, dmax, seed, dmin=1)
    return csr_from_degrees(deg, n, seed + 1, uniform_sources=uniform_sources, name=name)


# Named configurations (BASELINE.json configs)
CONFIGS = {
    # C1: n=1024, m=16384; corner rows 0 (deg 0), 1 (deg 1), 2 (deg 1024 = every vertex)
    "tiny": dict(n=1024, m=16384, sigma=1.0, dmax=512, corners=(0, 1, 1024), idx=1),
    # C2: ogbn-proteins-shaped, nnz = 2 x 39,561,252, lognormal sigma 0.9
    "proteins": dict(n=132534, m=79122504, sigma=0.9, dmax=7750, idx=2),
    # C3/C5: reddit-shaped, nnz = 114,615,892 (L9), lognormal sigma 1.2
    "reddit": dict(n=232965, m=114615892, sigma=1.2, dmax=21657, idx=3),
    # C4: rand-100K, 20K rows of degree 2000 + 80K rows of degree 100
    "rand100k": dict(n=100000, m=48000000, two_block=(20000, 2000, 80000, 100), idx=4),
}


def make_graph(name: str, uniform_sources: bool = False, scale: float = 1.0) -> Graph:
    """Build a named configuration graph.  `scale` < 1 shrinks n and m
    proportionally (tests only); scale = 1 is the BASELINE.json size."""
    c = CONFIGS[name]
    seed = SEED_BASE + c["idx"]
    if "two_block" in c:
        nh, dh, nl, dl = c["two_block"]
        if scale != 1.0:
            nh, nl = max(1, int(nh * scale)), max(1, int(nl * scale))
            dh, dl = max(1, min(int(dh * scale), nh + nl)), max(1, int(dl * scale))
        deg = degrees_two_block(nh, dh, nl, dl, seed)
    else:
        n, m = int(c["n"] * scale), int(c["m"] * scale)
        dmax = max(1, min(int(c["dmax"] * scale) if scale != 1.0 else c["dmax"], n))
        corners = c.get("corners", ())
        k = len(corners)
        rest = degrees_lognormal(n - k, m - sum(corners), c["sigma"], dmax, seed)
        deg = np.concatenate([np.asarray(corners, dtype=np.int64), rest])
    n = deg.size
    g = csr_from_degrees(deg, n, seed + 17, uniform_sources=uniform_sources,
                         name=name + ("-uniform" if uniform_sources else ""))
    return g


def feature_seed(graph_name: str) -> int:
    return SEED_BASE + CONFIGS[graph_name]["idx"] + 101


def to_bf16(x: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Storage conversion for the bf16-feature inputs (row f4): fp32 -> bf16 by
    round-to-nearest-even on the bit pattern (finite inputs).  Returns the
    uint16 bits (what the GPU side receives) and their exact fp32 decoding
    (what the oracle receives).  No method arithmetic: input preparation only."""
    b = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    bits = r.astype(np.uint16)
    dec = (bits.astype(np.uint32) << 16).view(np.float32)
    return bits, dec
