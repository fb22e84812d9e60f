"""GPU-vs-oracle parity for the edge cases the round-1 review named
(VERDICT r01 "What's weak" 2, 4), through the C ABI:

  * MLP with near-cancelling inputs: X_dst = -X + eps, every row holding a
    self-loop (s = x_v + x_dst_v = eps there) and some rows ONLY the
    self-loop -- the 1e-4 * sum_k |s_k W_k| bound (BASELINE north_star) must
    hold although |x_u W| is ~1e3 times larger than the message (the kernel
    forms s = x_u + x_v before the contraction, Fig. 3b);
    for the 3xTF32 product path and both ablations (FFMA, bf16 2-split);
  * edge softmax with score spreads > 100 inside a row (exp underflows fp32):
    DESIGN.md reading L15 -- |gpu - ref| <= 1e-4 * ref + 2^-126;
  * the fused GAT with integer scores of spread > 1000 (exact scores on both
    sides, so only the exp / normalisation differs);
  * fg_sddmm at F = 512 on an X wider than the segmentation threshold under
    CUDA-graph capture, with and without fg_graph_prepare (the op path never
    allocates or synchronises; prepared and unprepared results are bit-identical);
  * FG_TUNE_BALANCE_NNZ: shards whose automatic CTA-per-row threshold would
    differ from the whole graph's give bit-identical sums once the whole
    graph's edge count is set;
  * fg_dist_spmm / fg_dist_sddmm reject bad arguments BEFORE the all-gather
    (X_full untouched).
"""
import numpy as np
import pytest
import torch

import gen
import oracle
from helpers import check_close

pytestmark = pytest.mark.gpu
TOL = 1e-4
FLT_MIN = np.float64(2.0) ** -126


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.fixture(scope="module", autouse=True)
def _lib(cuda_ok):
    import paper_2008_11359_b200 as fgp
    fgp.lib()
    return fgp


def self_loop_graph(n, extra_deg, seed, only_self=200):
    """Every row v holds the self-loop v -> v; rows >= only_self also get
    `extra_deg` distinct random sources (ascending, no duplicates)."""
    rng = np.random.default_rng(seed)
    rows = []
    for v in range(n):
        if v < only_self:
            rows.append(np.array([v]))
        else:
            d = int(rng.integers(1, 2 * extra_deg))
            s = rng.choice(n, size=d, replace=False)
            rows.append(np.unique(np.concatenate([s, [v]])))
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([r.size for r in rows])
    return rp, np.concatenate(rows).astype(np.int32)


# ------------------------------------------------------------------ MLP cancellation
@pytest.mark.parametrize("impl", [0, 1, 2])
@pytest.mark.parametrize("d2", [32, 128])
@pytest.mark.parametrize("red", ["sum", "max"])
def test_mlp_near_cancelling_x_dst(impl, d2, red):
    import paper_2008_11359_b200 as fgp
    n, d1 = 3000, 8
    rp, ci = self_loop_graph(n, 40, 5 + d2)
    G = fgp.Graph(dev(rp), dev(ci))
    G.tune("mlp_impl", impl)
    X = gen.features((n, d1), 880, 0, gen.REAL)
    eps = gen.features((n, d1), 881, 0, gen.REAL) * np.float32(1e-3)
    Xd = (-X + eps).astype(np.float32)
    W = gen.features((d1, d2), 882, 0, gen.SCALED, scale=1 / np.sqrt(d1))
    ref, ab, _, _ = oracle.spmm(rp, ci, "mlp", red, X, W=W, X_dst=Xd)
    if red == "sum":
        out = fgp.spmm(G, "mlp", "sum", dev(X), W=dev(W), X_dst=dev(Xd)).cpu().numpy()
        check_close(out, ref, ab, TOL, f"mlp-sum cancelling impl={impl} d2={d2}")
        return
    out, au, ae = fgp.spmm(G, "mlp", "max", dev(X), W=dev(W), X_dst=dev(Xd), arg_u=True, arg_e=True)
    out, au, ae = out.cpu().numpy(), au.cpu().numpy(), ae.cpu().numpy()
    check_close(out, ref, ab, TOL, f"mlp-max cancelling impl={impl} d2={d2}")
    # argmax VALID: the oracle's message at the GPU's winning edge is within tolerance of the max
    X64, Xd64, W64 = X.astype(np.float64), Xd.astype(np.float64), W.astype(np.float64)
    for v in list(range(0, 200, 7)) + list(range(200, n, 37)):
        u = au[v]
        assert (ci[ae[v]] == u).all()
        z = ((X64[u] + Xd64[v][None, :]) * W64.T).sum(1)
        msg = np.maximum(z, 0.0)
        absz = (np.abs(X64[u] + Xd64[v][None, :]) * np.abs(W64.T)).sum(1)
        assert (np.abs(msg - ref[v]) <= TOL * (ab[v] + absz) + 1e-30).all()


# ------------------------------------------------------------------ softmax underflow (reading L15)
def softmax_close(got, ref):
    """DESIGN.md L15: relative 1e-4 per element, with an absolute floor of
    FLT_MIN = 2^-126 (fp32 carries no relative precision below it; exp of a
    score more than ~87 below its row's max underflows)."""
    got = got.astype(np.float64)
    return np.abs(got - ref) <= TOL * ref + FLT_MIN


@pytest.mark.parametrize("H", [1, 4, 8])
@pytest.mark.parametrize("spread", [100.0, 400.0])
def test_edge_softmax_wide_spread(H, spread):
    import paper_2008_11359_b200 as fgp
    g = gen.random_graph(3000, 120000, 91, sigma=1.6, n_empty=30)
    G = fgp.Graph(dev(g.row_ptr), dev(g.col_idx))
    S = (gen.features((g.nnz, H), 900 + H, 0, gen.UNIT) * np.float32(spread)).astype(np.float32)  # U[0,1) x spread
    out = fgp.edge_softmax(G, dev(S), H=H).cpu().numpy()
    ref = oracle.edge_softmax(g.row_ptr, S, H=H)
    assert np.isfinite(out).all() and (out >= 0).all()
    assert softmax_close(out, ref).all()
    # some weights really do underflow in this test (else it would not test the reading)
    assert (ref < FLT_MIN).any()
    rows = np.repeat(np.arange(g.n_dst), np.diff(g.row_ptr))
    sums = np.zeros((g.n_dst, H))
    np.add.at(sums, rows, out.astype(np.float64))
    nz = np.diff(g.row_ptr) > 0
    assert np.abs(sums[nz] - 1).max() <= TOL


@pytest.mark.parametrize("H,D", [(8, 32), (1, 64), (4, 16)])
def test_gat_fused_wide_spread_exact_scores(H, D):
    """Integer features: every score is an exact integer on both sides (|s| <=
    64 * D), spreads in a row reach hundreds, so the online softmax rescales
    through underflow; only exp / normalisation rounding remains."""
    import paper_2008_11359_b200 as fgp
    g = gen.random_graph(2000, 60000, 93, sigma=1.5, n_empty=20)
    G = fgp.Graph(dev(g.row_ptr), dev(g.col_idx))
    X = gen.features((g.n_src, H * D), 940, 0, gen.INT)
    Y = gen.features((g.n_dst, H * D), 941, 0, gen.INT)
    out = fgp.gat_attention(G, dev(X), dev(Y), H=H).cpu().numpy()
    ref, ab = oracle.gat(g.row_ptr, g.col_idx, X, Y, H=H)
    check_close(out, ref, ab + FLT_MIN, TOL, f"gat wide spread H={H} D={D}")
    s, _ = oracle.sddmm(g.row_ptr, g.col_idx, X, Y, H=H)
    deg = np.diff(g.row_ptr)
    rows = np.repeat(np.arange(g.n_dst), deg)
    spread = np.zeros((g.n_dst, H))
    mx = np.full((g.n_dst, H), -np.inf)
    mn = np.full((g.n_dst, H), np.inf)
    np.maximum.at(mx, rows, s)
    np.minimum.at(mn, rows, s)
    spread = (mx - mn)[deg > 1]
    assert spread.max() > 200   # the case under test does occur


# ------------------------------------------------------------------ CUDA-graph capture, prepare
def test_sddmm_capture_with_and_without_prepare():
    import paper_2008_11359_b200 as fgp
    n, m, F = 60000, 600000, 512                 # X = 123 MB > the 96 MB segmentation threshold
    g = gen.random_graph(n, m, 97, sigma=1.3, n_empty=100)
    Xh = gen.features((n, F), 950, 0, gen.REAL)
    X = dev(Xh)
    G = fgp.Graph(dev(g.row_ptr), dev(g.col_idx))
    before = G.info().device_bytes
    st = torch.cuda.Stream()
    ref_plain = fgp.sddmm(G, X, H=1, stream=st)    # not prepared: unsegmented traversal
    torch.cuda.synchronize()
    out = torch.empty_like(ref_plain)
    cg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(cg, stream=st):
        fgp.sddmm(G, X, H=1, out=out, stream=st)
    cg.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref_plain)
    assert G.info().device_bytes == before      # the op path allocated nothing
    G.prepare(F * 4)                             # the segmented table (synchronous)
    assert G.info().device_bytes > before
    out2 = torch.empty_like(ref_plain)
    cg2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(cg2, stream=st):
        fgp.sddmm(G, X, H=1, out=out2, stream=st)
    cg2.replay()
    torch.cuda.synchronize()
    assert torch.equal(out2, ref_plain)          # fg.h: prepared == unprepared, bit for bit
    rows = gen.permutation(n, 3)[:200]
    pos = oracle.edge_positions(g.row_ptr, rows)
    rs, rab = oracle.sddmm(g.row_ptr, g.col_idx, Xh, rows=rows)
    check_close(out2.cpu().numpy()[pos], rs, rab, TOL, "captured segmented sddmm")


# ------------------------------------------------------------------ FG_TUNE_BALANCE_NNZ
def test_balance_nnz_makes_shards_bit_identical():
    import paper_2008_11359_b200 as fgp
    from paper_2008_11359_b200.shard import make_shard
    # m = 20M, F = 512 (32-lane groups): the automatic threshold is
    # clamp(m / (SMs * 64), 1024, 4096) -- ~2100 for the whole graph, ~1050 for a
    # half -- and rows of degree 1000-3000 sit between them
    n = 12000
    deg = 1000 + (gen.permutation(n, 5) % 2000)
    g = gen.csr_from_degrees(deg.astype(np.int64), n, 77)
    X = dev(gen.features((n, 512), 960, 0, gen.REAL))
    G = fgp.Graph(dev(g.row_ptr), dev(g.col_idx))
    full = fgp.spmm(G, "copy_u", "sum", X)
    parts = []
    for r in range(2):
        sh = make_shard(g.row_ptr, g.col_idx, r, 2)
        L = fgp.Graph(dev(sh.row_ptr), dev(sh.col_idx), n_src=n)
        L.tune("balance_nnz", g.nnz)
        parts.append(fgp.spmm(L, "copy_u", "sum", X))
    assert torch.equal(torch.cat(parts), full)


# ------------------------------------------------------------------ dist ops: checks before the collective
def test_dist_ops_check_before_allgather():
    import paper_2008_11359_b200 as fgp
    c = fgp.Comm(fgp.comm_unique_id(), 1, 0)
    g = gen.random_graph(500, 8000, 98)
    G = fgp.Graph(dev(g.row_ptr), dev(g.col_idx))
    X_local = torch.ones(g.n_dst, 16, device="cuda")
    X_full = torch.full((g.n_dst, 16), 7.0, device="cuda")
    with pytest.raises(fgp.FGError) as e:   # H does not divide the width: FG_ESHAPE before any launch
        c.dist_spmm(G, [0, g.n_dst], "copy_u", "sum", X_local, X_full, H=3)
    L = fgp.lib()
    import ctypes
    off = np.array([0, g.n_dst], np.int64)
    bad_out = torch.empty(g.n_dst * 16 + 1, device="cuda")[1:]       # misaligned output
    st = L.fg_dist_spmm(G.handle, c.handle, ctypes.c_void_p(off.ctypes.data), 0, 0, 1, 16,
                        ctypes.c_void_p(X_local.data_ptr()), ctypes.c_void_p(X_full.data_ptr()), None, None, 0,
                        None, ctypes.c_void_p(bad_out.data_ptr()), None, None, None, 0, None)
    assert st == fgp.FG_EINVAL
    Y = torch.ones(g.n_dst, 16, device="cuda")
    s_out = torch.empty(g.nnz, 1, device="cuda")
    st = L.fg_dist_sddmm(G.handle, c.handle, ctypes.c_void_p(off.ctypes.data), 0, 3, 5,
                         ctypes.c_void_p(X_local.data_ptr()), ctypes.c_void_p(X_full.data_ptr()),
                         ctypes.c_void_p(Y.data_ptr()), ctypes.c_void_p(s_out.data_ptr()), None)
    assert st == fgp.FG_ESHAPE                                          # H*D = 15
    torch.cuda.synchronize()
    assert bool((X_full == 7.0).all())          # no all-gather ran
    assert e.value.status == fgp.FG_ESHAPE
    # a valid call does gather
    c.dist_spmm(G, [0, g.n_dst], "copy_u", "sum", X_local, X_full)
    torch.cuda.synchronize()
    assert bool((X_full == 1.0).all())
    c.close()
