"""GPU-vs-oracle parity through the C ABI (libfg.so), on seeded inputs from gen/.

Bar (BASELINE.json north_star):
  * integer / index outputs (argmax) bit-exact;
  * fp32 outputs |gpu - ref| <= 1e-4 * sum|terms| against the fp64 oracle;
  * integer-regime inputs: every output bit-exact (except softmax);
  * copy_u / u_mul_e max values bit-exact in every regime;
  * mlp argmax in the real regime checked as VALID.
Sizes span several CTAs / tiles, heavy (CTA-per-row) rows and ragged tails.
"""
import numpy as np
import pytest
import torch

import gen
import oracle
from helpers import check_close, csr_from_edges, tuned

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _lib(cuda_ok):
    import paper_2008_11359_b200 as fgp
    fgp.lib()
    return fgp


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


class G:
    """A graph on both sides: numpy arrays for the oracle, an fg handle for the GPU."""

    def __init__(self, row_ptr, col_idx, n_src=None, eid=None):
        import paper_2008_11359_b200 as fgp
        self.row_ptr = np.asarray(row_ptr, np.int64)
        self.col_idx = np.asarray(col_idx, np.int32)
        self.n_dst = self.row_ptr.size - 1
        self.n_src = self.n_dst if n_src is None else n_src
        self.nnz = int(self.row_ptr[-1])
        self.eid = None if eid is None else np.asarray(eid, np.int32)
        self.h = fgp.Graph(dev(self.row_ptr), dev(self.col_idx), n_src=self.n_src,
                           eid=None if eid is None else dev(self.eid))


def graph_of(g, eid=None):
    return G(g.row_ptr, g.col_idx, g.n_src, eid)


@pytest.fixture(scope="module")
def tiny():
    return graph_of(gen.make_graph("tiny"))


@pytest.fixture(scope="module")
def skewed():
    # 3000 rows, 120K edges, heavy rows up to 3000 (CTA-per-row path for every F), empty rows
    g = gen.random_graph(3000, 120000, 77, sigma=1.6, n_empty=50)
    return graph_of(g)


@pytest.fixture(scope="module")
def skewed_eid(skewed):
    return G(skewed.row_ptr, skewed.col_idx, skewed.n_src, eid=gen.permutation(skewed.nnz, 13).astype(np.int32))


def feats(shape, seed, regime, lo=-8, hi=8):
    return gen.features(shape, seed, 0, regime, lo=lo, hi=hi)


# ------------------------------------------------------------------ copy_u
@pytest.mark.parametrize("F", [4, 8, 16, 32, 48, 128, 200, 256, 512, 640])
@pytest.mark.parametrize("regime", [gen.REAL, gen.INT])
def test_copy_u_sum(skewed, F, regime):
    import paper_2008_11359_b200 as fgp
    X = feats((skewed.n_src, F), 100 + F, regime)
    out = fgp.spmm(skewed.h, "copy_u", "sum", dev(X)).cpu().numpy()
    ref, ab, _, _ = oracle.spmm(skewed.row_ptr, skewed.col_idx, "copy_u", "sum", X)
    if regime == gen.INT:
        assert np.array_equal(out.astype(np.float64), ref)
    else:
        check_close(out, ref, ab, TOL, f"copy_u-sum F={F}")


@pytest.mark.parametrize("F", [4, 16, 32, 64, 128, 384, 512, 1024])
@pytest.mark.parametrize("regime", [gen.REAL, gen.INT])
def test_copy_u_max(skewed, F, regime):
    import paper_2008_11359_b200 as fgp
    X = feats((skewed.n_src, F), 200 + F, regime, lo=-3, hi=3)   # INT: heavy ties
    out, au, ae = fgp.spmm(skewed.h, "copy_u", "max", dev(X), arg_u=True, arg_e=True)
    ref, _, rau, rae = oracle.spmm(skewed.row_ptr, skewed.col_idx, "copy_u", "max", X)
    assert np.array_equal(out.cpu().numpy().astype(np.float64), ref)
    assert np.array_equal(au.cpu().numpy(), rau)
    assert np.array_equal(ae.cpu().numpy(), rae)


@pytest.mark.parametrize("F", [4, 32, 128, 512])
@pytest.mark.parametrize("regime", [gen.REAL, gen.INT])
def test_copy_u_min(skewed, F, regime):
    """row f4: min = first-wins argmin, bit-exact with the oracle."""
    import paper_2008_11359_b200 as fgp
    X = feats((skewed.n_src, F), 250 + F, regime, lo=-3, hi=3)
    out, au, ae = fgp.spmm(skewed.h, "copy_u", "min", dev(X), arg_u=True, arg_e=True)
    ref, _, rau, rae = oracle.spmm(skewed.row_ptr, skewed.col_idx, "copy_u", "min", X)
    assert np.array_equal(out.cpu().numpy().astype(np.float64), ref)
    assert np.array_equal(au.cpu().numpy(), rau)
    assert np.array_equal(ae.cpu().numpy(), rae)


@pytest.mark.parametrize("F", [4, 32, 128, 512])
@pytest.mark.parametrize("regime", [gen.REAL, gen.INT])
def test_copy_u_mean(skewed, F, regime):
    """row f4: mean = sum / |N(v)|.  INT regime: the fp32 sum is exact, so the one
    IEEE division gives exactly fp32(oracle)."""
    import paper_2008_11359_b200 as fgp
    X = feats((skewed.n_src, F), 260 + F, regime)
    out = fgp.spmm(skewed.h, "copy_u", "mean", dev(X)).cpu().numpy()
    ref, ab, _, _ = oracle.spmm(skewed.row_ptr, skewed.col_idx, "copy_u", "mean", X)
    if regime == gen.INT:
        assert np.array_equal(out, ref.astype(np.float32))
    else:
        check_close(out, ref, ab, TOL, f"copy_u-mean F={F}")


def test_tiny_config_all_ops(tiny):
    """BASELINE.json configs[0]: tiny graph, F=16, copy_u sum/max + u_dot_v."""
    import paper_2008_11359_b200 as fgp
    F = 16
    X = feats((tiny.n_src, F), 1, gen.REAL)
    out = fgp.spmm(tiny.h, "copy_u", "sum", dev(X)).cpu().numpy()
    ref, ab, _, _ = oracle.spmm(tiny.row_ptr, tiny.col_idx, "copy_u", "sum", X)
    check_close(out, ref, ab, TOL, "tiny copy_u-sum")
    out, au, ae = fgp.spmm(tiny.h, "copy_u", "max", dev(X), arg_u=True, arg_e=True)
    ref, _, rau, rae = oracle.spmm(tiny.row_ptr, tiny.col_idx, "copy_u", "max", X)
    assert np.array_equal(out.cpu().numpy().astype(np.float64), ref)
    assert np.array_equal(au.cpu().numpy(), rau) and np.array_equal(ae.cpu().numpy(), rae)
    s = fgp.sddmm(tiny.h, dev(X)).cpu().numpy()
    ref, ab = oracle.sddmm(tiny.row_ptr, tiny.col_idx, X)
    check_close(s, ref, ab, TOL, "tiny u_dot_v")


# ------------------------------------------------------------------ u_mul_e
@pytest.mark.parametrize("H,D", [(1, 4), (1, 128), (2, 2), (8, 2), (4, 4), (8, 32), (8, 64), (3, 12)])
@pytest.mark.parametrize("red", ["sum", "max", "min", "mean"])
@pytest.mark.parametrize("use_eid", [False, True])
def test_u_mul_e(skewed, skewed_eid, H, D, red, use_eid):
    import paper_2008_11359_b200 as fgp
    g = skewed_eid if use_eid else skewed
    F = H * D
    X = feats((g.n_src, F), 300 + F, gen.REAL)
    E = gen.features((g.nnz, H), 301, 1, gen.UNIT)
    ref, ab, rau, rae = oracle.spmm(g.row_ptr, g.col_idx, "u_mul_e", red, X, H=H, E=E, eid=g.eid)
    if red in ("sum", "mean"):
        out = fgp.spmm(g.h, "u_mul_e", red, dev(X), H=H, E=dev(E)).cpu().numpy()
        check_close(out, ref, ab, TOL, f"u_mul_e-{red} H={H} D={D}")
    else:
        out, au, ae = fgp.spmm(g.h, "u_mul_e", red, dev(X), H=H, E=dev(E), arg_u=True, arg_e=True)
        assert np.array_equal(out.cpu().numpy().astype(np.float64), ref)
        assert np.array_equal(au.cpu().numpy(), rau)
        assert np.array_equal(ae.cpu().numpy(), rae)


@pytest.mark.parametrize("H,D", [(1, 4), (2, 2), (8, 32), (3, 12), (4, 3), (1, 128)])
@pytest.mark.parametrize("red", ["sum", "max", "min", "mean"])
@pytest.mark.parametrize("use_eid", [False, True])
def test_u_add_e(skewed, skewed_eid, H, D, red, use_eid):
    """row f4: phi = x_u + e (E [nnz][H] broadcast over D)."""
    import paper_2008_11359_b200 as fgp
    g = skewed_eid if use_eid else skewed
    F = H * D
    X = feats((g.n_src, F), 320 + F, gen.REAL)
    E = gen.features((g.nnz, H), 321, 1, gen.REAL)
    ref, ab, rau, rae = oracle.spmm(g.row_ptr, g.col_idx, "u_add_e", red, X, H=H, E=E, eid=g.eid)
    if red in ("sum", "mean"):
        out = fgp.spmm(g.h, "u_add_e", red, dev(X), H=H, E=dev(E)).cpu().numpy()
        check_close(out, ref, ab, TOL, f"u_add_e-{red} H={H} D={D}")
    else:
        out, au, ae = fgp.spmm(g.h, "u_add_e", red, dev(X), H=H, E=dev(E), arg_u=True, arg_e=True)
        assert np.array_equal(out.cpu().numpy().astype(np.float64), ref)
        assert np.array_equal(au.cpu().numpy(), rau)
        assert np.array_equal(ae.cpu().numpy(), rae)


@pytest.mark.parametrize("F", [4, 32, 128, 260, 512])
@pytest.mark.parametrize("red", ["sum", "max", "min", "mean"])
@pytest.mark.parametrize("use_eid", [False, True])
def test_copy_e(skewed, skewed_eid, F, red, use_eid):
    """row f4: phi = the edge's own feature row E[eid] ([nnz][F])."""
    import paper_2008_11359_b200 as fgp
    g = skewed_eid if use_eid else skewed
    E = gen.features((g.nnz, F), 330 + F, 0, gen.INT if red in ("max", "min") else gen.REAL, lo=-3, hi=3)
    ref, ab, rau, rae = oracle.spmm(g.row_ptr, g.col_idx, "copy_e", red, None, E=E, eid=g.eid)
    if red in ("sum", "mean"):
        out = fgp.spmm(g.h, "copy_e", red, None, E=dev(E)).cpu().numpy()
        check_close(out, ref, ab, TOL, f"copy_e-{red} F={F}")
    else:
        out, au, ae = fgp.spmm(g.h, "copy_e", red, None, E=dev(E), arg_u=True, arg_e=True)
        assert np.array_equal(out.cpu().numpy().astype(np.float64), ref)
        assert np.array_equal(au.cpu().numpy(), rau)
        assert np.array_equal(ae.cpu().numpy(), rae)


def test_u_mul_e_int_regime_exact(skewed):
    import paper_2008_11359_b200 as fgp
    H, D = 8, 32
    X = feats((skewed.n_src, H * D), 311, gen.INT)
    E = gen.features((skewed.nnz, H), 312, 1, gen.INT, lo=0, hi=4)
    out = fgp.spmm(skewed.h, "u_mul_e", "sum", dev(X), H=H, E=dev(E)).cpu().numpy()
    ref, _, _, _ = oracle.spmm(skewed.row_ptr, skewed.col_idx, "u_mul_e", "sum", X, H=H, E=E)
    assert np.array_equal(out.astype(np.float64), ref)


# ------------------------------------------------------------------ mlp
@pytest.mark.parametrize("d2", [16, 128, 256])
@pytest.mark.parametrize("red", ["max", "sum"])
def test_mlp_int_exact(skewed, d2, red):
    import paper_2008_11359_b200 as fgp
    d1 = 8
    X = feats((skewed.n_src, d1), 400, gen.INT)
    W = gen.features((d1, d2), 401, 1, gen.INT, lo=-4, hi=4)
    ref, _, rau, rae = oracle.spmm(skewed.row_ptr, skewed.col_idx, "mlp", red, X, W=W)
    if red == "max":
        out, au, ae = fgp.spmm(skewed.h, "mlp", "max", dev(X), W=dev(W), arg_u=True, arg_e=True)
        assert np.array_equal(au.cpu().numpy(), rau)
        assert np.array_equal(ae.cpu().numpy(), rae)
    else:
        out = fgp.spmm(skewed.h, "mlp", "sum", dev(X), W=dev(W))
    assert np.array_equal(out.cpu().numpy().astype(np.float64), ref)


@pytest.mark.parametrize("d2", [32, 128])
@pytest.mark.parametrize("red", ["max", "sum"])
def test_mlp_real(skewed, d2, red):
    import paper_2008_11359_b200 as fgp
    d1 = 8
    X = feats((skewed.n_src, d1), 410, gen.REAL)
    W = gen.features((d1, d2), 411, 1, gen.SCALED, scale=1 / np.sqrt(d1))
    ref, ab, _, _ = oracle.spmm(skewed.row_ptr, skewed.col_idx, "mlp", red, X, W=W)
    if red == "sum":
        out = fgp.spmm(skewed.h, "mlp", "sum", dev(X), W=dev(W)).cpu().numpy()
        check_close(out, ref, ab, TOL, f"mlp-sum d2={d2}")
        return
    out, au, ae = fgp.spmm(skewed.h, "mlp", "max", dev(X), W=dev(W), arg_u=True, arg_e=True)
    out, au, ae = out.cpu().numpy(), au.cpu().numpy(), ae.cpu().numpy()
    check_close(out, ref, ab, TOL, f"mlp-max d2={d2}")
    # argmax VALID: the oracle's message at the GPU's winning edge is within tolerance of the max
    Xd, Wd = X.astype(np.float64), W.astype(np.float64)
    deg = np.diff(skewed.row_ptr)
    for v in np.flatnonzero(deg)[::7]:
        u = au[v]
        assert (skewed.col_idx[ae[v]] == u).all()
        msg = np.maximum(((Xd[u] + Xd[v][None, :]) * Wd.T).sum(1), 0.0)
        assert (np.abs(msg - ref[v]) <= TOL * ab[v] + 1e-30).all()


def test_mlp_separate_x_dst():
    import paper_2008_11359_b200 as fgp
    g = graph_of(gen.random_graph(500, 8000, 5, n_empty=5))
    X = feats((g.n_src, 8), 420, gen.INT)
    Xd = feats((g.n_dst, 8), 421, gen.INT)
    W = gen.features((8, 64), 422, 1, gen.INT, lo=-4, hi=4)
    out, au, _ = fgp.spmm(g.h, "mlp", "max", dev(X), W=dev(W), X_dst=dev(Xd), arg_u=True)
    ref, _, rau, _ = oracle.spmm(g.row_ptr, g.col_idx, "mlp", "max", X, W=W, X_dst=Xd)
    assert np.array_equal(out.cpu().numpy().astype(np.float64), ref)
    assert np.array_equal(au.cpu().numpy(), rau)


# ------------------------------------------------------------------ sddmm
@pytest.mark.parametrize("H,D", [(1, 4), (1, 16), (1, 48), (1, 128), (1, 512), (1, 1024), (2, 4), (8, 4),
                                 (8, 32), (4, 64), (2, 256), (8, 8), (12, 32), (6, 64), (3, 128), (24, 16),
                                 (5, 64)])
@pytest.mark.parametrize("use_eid", [False, True])
def test_sddmm(skewed, skewed_eid, H, D, use_eid):
    import paper_2008_11359_b200 as fgp
    g = skewed_eid if use_eid else skewed
    F = H * D
    X = feats((g.n_src, F), 500 + F, gen.REAL)
    Y = feats((g.n_dst, F), 501 + F, gen.REAL)
    out = fgp.sddmm(g.h, dev(X), dev(Y), H=H).cpu().numpy()
    ref, ab = oracle.sddmm(g.row_ptr, g.col_idx, X, Y, H=H)   # CSR order
    pos = np.arange(g.nnz) if g.eid is None else g.eid
    check_close(out[pos], ref, ab, TOL, f"u_dot_v H={H} D={D}")


@pytest.mark.parametrize("op", ["u_add_v", "u_sub_v", "u_mul_v"])
@pytest.mark.parametrize("F", [4, 12, 128, 516])
@pytest.mark.parametrize("use_eid", [False, True])
def test_sddmm_binary(skewed, skewed_eid, op, F, use_eid):
    """row f4: elementwise u_OP_v; one IEEE op per element, so the kernel equals
    fp32(oracle) exactly."""
    import paper_2008_11359_b200 as fgp
    g = skewed_eid if use_eid else skewed
    X = feats((g.n_src, F), 400 + F, gen.REAL)
    Y = feats((g.n_dst, F), 401 + F, gen.REAL)
    out = fgp.sddmm(g.h, dev(X), dev(Y), op=op).cpu().numpy()
    ref, _ = oracle.sddmm_binary(g.row_ptr, g.col_idx, op, X, Y)
    pos = np.arange(g.nnz) if g.eid is None else g.eid
    assert np.array_equal(out[pos], ref.astype(np.float32))


def test_sddmm_int_exact(skewed):
    import paper_2008_11359_b200 as fgp
    H, D = 8, 32
    X = feats((skewed.n_src, H * D), 510, gen.INT)
    out = fgp.sddmm(skewed.h, dev(X), H=H).cpu().numpy()
    ref, _ = oracle.sddmm(skewed.row_ptr, skewed.col_idx, X, H=H)
    assert np.array_equal(out.astype(np.float64), ref)


# ------------------------------------------------------------------ edge softmax
@pytest.mark.parametrize("H", [1, 2, 4, 8, 16, 3])
@pytest.mark.parametrize("use_eid", [False, True])
def test_edge_softmax(skewed, skewed_eid, H, use_eid):
    import paper_2008_11359_b200 as fgp
    g = skewed_eid if use_eid else skewed
    S = gen.features((g.nnz, H), 600 + H, 0, gen.REAL) * 8
    out = fgp.edge_softmax(g.h, dev(S), H=H).cpu().numpy()
    ref = oracle.edge_softmax(g.row_ptr, S, H=H, eid=g.eid)   # CSR order
    pos = np.arange(g.nnz) if g.eid is None else g.eid
    got = out[pos].astype(np.float64)
    assert (np.abs(got - ref) <= TOL * ref).all()
    rows = np.repeat(np.arange(g.n_dst), np.diff(g.row_ptr))
    sums = np.zeros((g.n_dst, H))
    np.add.at(sums, rows, got)
    nz = np.diff(g.row_ptr) > 0
    assert np.abs(sums[nz] - 1).max() <= TOL
    # in place
    St = dev(S)
    fgp.edge_softmax(g.h, St, H=H, out=St)
    assert np.array_equal(St.cpu().numpy(), out)


@pytest.mark.parametrize("H", [4, 8, 32])
def test_edge_softmax_staging_boundaries(H):
    """Row-length edge cases around the 8 KiB-of-scores mark (cap = 2048 / H
    edges): rows of degree cap - 1, cap, cap + 1, a run of small rows, empty
    rows, and a row several caps long."""
    import paper_2008_11359_b200 as fgp
    cap = 8 * 1024 // (4 * H)
    rng = np.random.default_rng(H)
    degs = [cap - 1, 0, cap, 1, cap + 1, 0, 0, 3 * cap + 7] + list(rng.integers(0, 40, 600)) + [cap, 2]
    rp = np.concatenate([[0], np.cumsum(degs)]).astype(np.int64)
    ci = np.concatenate([np.sort(rng.choice(4 * cap, size=d, replace=False)) for d in degs]).astype(np.int32)
    g = G(rp, ci, n_src=4 * cap)
    S = gen.features((g.nnz, H), 640 + H, 0, gen.REAL) * 8
    out = fgp.edge_softmax(g.h, dev(S), H=H).cpu().numpy().astype(np.float64)
    ref = oracle.edge_softmax(g.row_ptr, S, H=H)
    assert (np.abs(out - ref) <= TOL * ref).all()


def test_edge_softmax_special_values(skewed):
    import paper_2008_11359_b200 as fgp
    H = 4
    S = np.full((skewed.nnz, H), 0.75, np.float32)
    out = fgp.edge_softmax(skewed.h, dev(S), H=H).cpu().numpy()
    deg = np.diff(skewed.row_ptr)
    rows = np.repeat(np.arange(skewed.n_dst), deg)
    expect = (np.float32(1.0) / deg[rows].astype(np.float32))[:, None]
    assert np.array_equal(out, np.broadcast_to(expect, out.shape))   # constant -> 1/deg (correctly rounded)


# ------------------------------------------------------------------ chain (GAT layer, config 3 shape at small size)
def test_gat_layer_chain(skewed):
    """sddmm -> edge_softmax -> u_mul_e, each op checked in isolation on the
    ORACLE's fp32-rounded intermediates (no compounding through
    exp; no oracle input comes from the CUDA path), then the GPU chain end to
    end against the fused-layer definition oracle.gat."""
    import paper_2008_11359_b200 as fgp
    H, D = 8, 32
    X = feats((skewed.n_src, H * D), 700, gen.REAL) * 0.25
    Xt = dev(X)
    ref_s, ab_s = oracle.sddmm(skewed.row_ptr, skewed.col_idx, X, H=H)
    s32 = ref_s.astype(np.float32)
    ref_a = oracle.edge_softmax(skewed.row_ptr, s32, H=H)
    a32 = ref_a.astype(np.float32)
    ref_o, ab_o, _, _ = oracle.spmm(skewed.row_ptr, skewed.col_idx, "u_mul_e", "sum", X, H=H, E=a32)
    s = fgp.sddmm(skewed.h, Xt, H=H)
    check_close(s.cpu().numpy(), ref_s, ab_s, TOL, "gat sddmm")
    a = fgp.edge_softmax(skewed.h, dev(s32), H=H).cpu().numpy()
    assert (np.abs(a - ref_a) <= TOL * ref_a).all()
    out = fgp.spmm(skewed.h, "u_mul_e", "sum", Xt, H=H, E=dev(a32)).cpu().numpy()
    check_close(out, ref_o, ab_o, TOL, "gat aggregation")
    chain = fgp.spmm(skewed.h, "u_mul_e", "sum", Xt, H=H, E=fgp.edge_softmax(skewed.h, s, H=H)).cpu().numpy()
    ref_g, ab_g = oracle.gat(skewed.row_ptr, skewed.col_idx, X, H=H)
    check_close(chain, ref_g, ab_g, TOL, "gat chain end to end")


# ------------------------------------------------------------------ degenerate graphs and ABI behaviour
@pytest.mark.parametrize("case", ["n1_m0", "all_empty", "one_row_all_edges", "self_loop", "n_src_ne_n_dst"])
def test_degenerate(case):
    import paper_2008_11359_b200 as fgp
    if case == "n1_m0":
        g = G(np.array([0, 0]), np.zeros(0, np.int32))
    elif case == "all_empty":
        g = G(np.zeros(65, np.int64), np.zeros(0, np.int32))
    elif case == "one_row_all_edges":
        n = 5000
        rp = np.zeros(n + 1, np.int64)
        rp[1:] = n
        g = G(rp, np.arange(n, dtype=np.int32))
    elif case == "self_loop":
        rp, ci = csr_from_edges(3, [[0, 0], [1, 1], [2, 2], [0, 2]])
        g = G(rp, ci)
    else:
        rp, ci = csr_from_edges(4, [[0, 1], [5, 1], [6, 3], [2, 0]], n_src=7)
        g = G(rp, ci, n_src=7)
    for F in (4, 32, 512):
        X = feats((g.n_src, F), 800 + F, gen.REAL)
        out = torch.full((g.n_dst, F), float("nan"), device="cuda")
        fgp.spmm(g.h, "copy_u", "sum", dev(X), out=out)
        ref, ab, _, _ = oracle.spmm(g.row_ptr, g.col_idx, "copy_u", "sum", X)
        check_close(out.cpu().numpy(), ref, ab, TOL, f"{case} sum F={F}")
        out = torch.full((g.n_dst, F), float("nan"), device="cuda")
        au = torch.full((g.n_dst, F), 7, dtype=torch.int32, device="cuda")
        fgp.spmm(g.h, "copy_u", "max", dev(X), out=out, arg_u=au)
        ref, _, rau, _ = oracle.spmm(g.row_ptr, g.col_idx, "copy_u", "max", X)
        assert np.array_equal(out.cpu().numpy().astype(np.float64), ref)
        assert np.array_equal(au.cpu().numpy(), rau)
        if g.nnz:
            Y = feats((g.n_dst, F), 900 + F, gen.REAL)
            s = fgp.sddmm(g.h, dev(X), dev(Y)).cpu().numpy()
            ref, ab = oracle.sddmm(g.row_ptr, g.col_idx, X, Y)
            check_close(s, ref, ab, TOL, f"{case} sddmm F={F}")


def test_determinism(skewed):
    import paper_2008_11359_b200 as fgp
    X = dev(feats((skewed.n_src, 256), 950, gen.REAL))
    a = fgp.spmm(skewed.h, "copy_u", "sum", X)
    b = fgp.spmm(skewed.h, "copy_u", "sum", X)
    assert torch.equal(a, b)
    s1, s2 = fgp.sddmm(skewed.h, X, H=8), fgp.sddmm(skewed.h, X, H=8)
    assert torch.equal(s1, s2)


def test_abi_errors_on_device(skewed):
    import paper_2008_11359_b200 as fgp
    from paper_2008_11359_b200.fg import FGError, FG_EINVAL, FG_ESHAPE, FG_EGRAPH
    X = torch.zeros((skewed.n_src * 8 + 1,), device="cuda")
    with pytest.raises(FGError) as ei:   # misaligned X
        fgp.spmm(skewed.h, "copy_u", "sum", X[1:].view(skewed.n_src, 8))
    assert ei.value.status == FG_EINVAL
    with pytest.raises(FGError) as ei:   # F % 4 != 0
        fgp.spmm(skewed.h, "copy_u", "sum", torch.zeros((skewed.n_src, 6), device="cuda"))
    assert ei.value.status == FG_ESHAPE
    with pytest.raises(FGError) as ei:   # arg with sum
        fgp.spmm(skewed.h, "copy_u", "sum", torch.zeros((skewed.n_src, 8), device="cuda"), arg_u=True)
    assert ei.value.status == FG_EINVAL
    with pytest.raises(FGError) as ei:   # arg with mean
        fgp.spmm(skewed.h, "copy_u", "mean", torch.zeros((skewed.n_src, 8), device="cuda"), arg_u=True)
    assert ei.value.status == FG_EINVAL
    with pytest.raises(FGError) as ei:   # mlp supports sum / max only
        fgp.spmm(skewed.h, "mlp", "min", torch.zeros((skewed.n_src, 8), device="cuda"),
                 W=torch.zeros((8, 16), device="cuda"))
    assert ei.value.status == fgp.fg.FG_EUNSUPPORTED
    out = torch.full((skewed.n_dst, 8), 3.0, device="cuda")
    with pytest.raises(FGError):
        fgp.spmm(skewed.h, "copy_u", "sum", torch.zeros((skewed.n_src, 6), device="cuda"), out=out)
    assert (out == 3.0).all()   # untouched on error
    # CSR validation
    rp = np.array([0, 2, 3], np.int64)
    for ci, why in [(np.array([1, 0, 0], np.int32), "unsorted"), (np.array([0, 5, 1], np.int32), "range")]:
        with pytest.raises(FGError) as ei:
            fgp.Graph(dev(rp), dev(ci), n_src=2)
        assert ei.value.status == FG_EGRAPH, why
    with pytest.raises(FGError) as ei:
        fgp.Graph(dev(np.array([0, 1, 2], np.int64)), dev(np.array([0, 1], np.int32)),
                  eid=dev(np.array([1, 1], np.int32)))
    assert ei.value.status == FG_EGRAPH


# ------------------------------------------------------------------ L2 feature-dimension tiling paths
@pytest.mark.parametrize("F", [128, 512, 1024])
def test_l2_column_tiling(skewed, F):
    """Force the column-tiled (multi-pass) paths with a tiny L2 budget: copy_u
    sum/max and H=1 u_dot_v must still match the oracle (max bit-exact)."""
    with tuned(skewed.h, l2_tile_mb=1, sddmm_l2_tile=1):
        _l2_column_tiling(skewed, F)


def _l2_column_tiling(skewed, F):
    import paper_2008_11359_b200 as fgp
    X = feats((skewed.n_src, F), 960 + F, gen.REAL)
    Y = feats((skewed.n_dst, F), 961 + F, gen.REAL)
    out = fgp.spmm(skewed.h, "copy_u", "sum", dev(X)).cpu().numpy()
    ref, ab, _, _ = oracle.spmm(skewed.row_ptr, skewed.col_idx, "copy_u", "sum", X)
    check_close(out, ref, ab, TOL, f"tiled copy_u-sum F={F}")
    mx, au, ae = fgp.spmm(skewed.h, "copy_u", "max", dev(X), arg_u=True, arg_e=True)
    ref, _, rau, rae = oracle.spmm(skewed.row_ptr, skewed.col_idx, "copy_u", "max", X)
    assert np.array_equal(mx.cpu().numpy().astype(np.float64), ref)
    assert np.array_equal(au.cpu().numpy(), rau) and np.array_equal(ae.cpu().numpy(), rae)
    mn, au = fgp.spmm(skewed.h, "copy_u", "min", dev(X), arg_u=True)[:2]
    ref, _, rau, _ = oracle.spmm(skewed.row_ptr, skewed.col_idx, "copy_u", "min", X)
    assert np.array_equal(mn.cpu().numpy().astype(np.float64), ref) and np.array_equal(au.cpu().numpy(), rau)
    me = fgp.spmm(skewed.h, "copy_u", "mean", dev(X)).cpu().numpy()
    ref, ab, _, _ = oracle.spmm(skewed.row_ptr, skewed.col_idx, "copy_u", "mean", X)
    check_close(me, ref, ab, TOL, f"tiled copy_u-mean F={F}")
    s = fgp.sddmm(skewed.h, dev(X), dev(Y)).cpu().numpy()
    ref, ab = oracle.sddmm(skewed.row_ptr, skewed.col_idx, X, Y)
    check_close(s, ref, ab, TOL, f"tiled u_dot_v F={F}")
    skewed.h.tune("l2_tile_mb", 0)
    s0 = fgp.sddmm(skewed.h, dev(X), dev(Y)).cpu().numpy()
    check_close(s0, ref, ab, TOL, f"untiled u_dot_v F={F}")


@pytest.mark.parametrize("H,D", [(1, 512), (1, 128), (8, 32), (2, 4)])
@pytest.mark.parametrize("use_eid", [False, True])
def test_sddmm_source_segmented(skewed, skewed_eid, H, D, use_eid):
    """Row f3: force the source-segmented persistent SDDMM (1 MB segments ->
    several segments even on the small test graph, tables built by
    fg_graph_prepare) and compare with the oracle."""
    g = skewed_eid if use_eid else skewed
    with tuned(g.h, sddmm_seg_mb=1, sddmm_seg_min_mb=0):
        g.h.prepare(H * D * 4)
        g.h.prepare(H * D * 2)
        _sddmm_source_segmented(g, H, D)


def _sddmm_source_segmented(g, H, D):
    import paper_2008_11359_b200 as fgp
    X = feats((g.n_src, H * D), 980 + D, gen.REAL)
    Y = feats((g.n_dst, H * D), 981 + D, gen.REAL)
    out = fgp.sddmm(g.h, dev(X), dev(Y), H=H).cpu().numpy()
    ref, ab = oracle.sddmm(g.row_ptr, g.col_idx, X, Y, H=H)
    pos = np.arange(g.nnz) if g.eid is None else g.eid
    check_close(out[pos], ref, ab, TOL, f"segmented u_dot_v H={H} D={D}")
    with tuned(g.h, sddmm_persist=1):             # one CTA per SM: every group walks many units
        out1 = fgp.sddmm(g.h, dev(X), dev(Y), H=H).cpu().numpy()
    assert np.array_equal(out1, out)              # same per-edge arithmetic, any schedule
    with tuned(g.h, sddmm_seg_mb=0):              # unsegmented: still bit-identical (fg.h fg_graph_prepare)
        out0 = fgp.sddmm(g.h, dev(X), dev(Y), H=H).cpu().numpy()
    assert np.array_equal(out0, out)
    if H * D % 8 == 0:   # the bf16 pair kernel on the same segmented units
        xb, xd = gen.to_bf16(X)
        yb, yd = gen.to_bf16(Y)
        outb = fgp.sddmm(g.h, bf16_dev(xb), bf16_dev(yb), H=H).cpu().numpy()
        rb, rbb = oracle.sddmm(g.row_ptr, g.col_idx, xd, yd, H=H)
        check_close(outb[pos], rb, rbb, TOL, f"segmented bf16 u_dot_v H={H} D={D}")


@pytest.mark.parametrize("H,D", [(8, 32), (1, 512), (2, 4), (4, 64), (8, 16)])
@pytest.mark.parametrize("use_eid", [False, True])
@pytest.mark.parametrize("heavy", [0, 64])
def test_spmm_u_mul_e_source_segmented(skewed, skewed_eid, H, D, use_eid, heavy):
    """Row f3 / a2: force the source-segmented u_mul_e-sum passes (1 MB segments
    -> several segments on the small graph; bounds built by fg_graph_prepare),
    also with most rows split CTA-per-row (heavy = 64), and compare with the
    oracle.  Rows summed group-per-row keep the CSR order: bit-identical to the
    unsegmented kernel (include/fg.h fg_graph_prepare)."""
    import paper_2008_11359_b200 as fgp
    g = skewed_eid if use_eid else skewed
    F = H * D
    X = feats((g.n_src, F), 990 + F, gen.REAL)
    E = gen.features((g.nnz, H), 991, 1, gen.UNIT)
    ref, ab, _, _ = oracle.spmm(g.row_ptr, g.col_idx, "u_mul_e", "sum", X, H=H, E=E, eid=g.eid)
    with tuned(g.h, spmm_seg_mb=1, sddmm_seg_min_mb=0, spmm_heavy_deg=heavy):
        g.h.prepare(F * 4)
        out = torch.full((g.n_dst, F), float("nan"), device="cuda")
        fgp.spmm(g.h, "u_mul_e", "sum", dev(X), H=H, E=dev(E), out=out)
        out = out.cpu().numpy()
        check_close(out, ref, ab, TOL, f"segmented u_mul_e-sum H={H} D={D}")
        again = fgp.spmm(g.h, "u_mul_e", "sum", dev(X), H=H, E=dev(E)).cpu().numpy()
        assert np.array_equal(again, out)         # deterministic: fixed segment order, no atomics
        with tuned(g.h, spmm_seg_mb=0):
            plain = fgp.spmm(g.h, "u_mul_e", "sum", dev(X), H=H, E=dev(E)).cpu().numpy()
    deg = np.diff(g.row_ptr)
    light = deg < (heavy if heavy else 1024)      # the automatic threshold is >= 1024
    assert np.array_equal(out[light], plain[light])
    # integer regime: every partial sum exact, so every row (heavy ones too) is bit-exact
    Xi = feats((g.n_src, F), 992 + F, gen.INT)
    Ei = gen.features((g.nnz, H), 993, 1, gen.INT, lo=0, hi=4)
    refi, _, _, _ = oracle.spmm(g.row_ptr, g.col_idx, "u_mul_e", "sum", Xi, H=H, E=Ei, eid=g.eid)
    with tuned(g.h, spmm_seg_mb=1, sddmm_seg_min_mb=0, spmm_heavy_deg=heavy):
        outi = fgp.spmm(g.h, "u_mul_e", "sum", dev(Xi), H=H, E=dev(Ei)).cpu().numpy()
    assert np.array_equal(outi.astype(np.float64), refi)


@pytest.mark.parametrize("F", [260, 384, 512, 200, 128, 100])
@pytest.mark.parametrize("use_eid", [False, True])
def test_sddmm_pipelined_and_hilbert(skewed, skewed_eid, F, use_eid):
    """a4 / f3: the software-pipelined wide-row H=1 kernel (every variant) and the
    Hilbert-ordered 2D unit tables against the oracle, and bit for
    bit against the plain segment-major kernel (same lane partition and
    reduction tree; only the schedule differs)."""
    import paper_2008_11359_b200 as fgp
    g = skewed_eid if use_eid else skewed
    X = feats((g.n_src, F), 1200 + F, gen.REAL)
    Y = feats((g.n_dst, F), 1201 + F, gen.REAL)
    ref, ab = oracle.sddmm(g.row_ptr, g.col_idx, X, Y)
    pos = np.arange(g.nnz) if g.eid is None else g.eid
    with tuned(g.h, sddmm_pipe=0):
        plain = fgp.sddmm(g.h, dev(X), dev(Y)).cpu().numpy()
    check_close(plain[pos], ref, ab, TOL, f"u_dot_v F={F}")
    for pipe in (1, 2, 3, 4, 5, 6, 7, -1):
        with tuned(g.h, sddmm_pipe=pipe):
            out = fgp.sddmm(g.h, dev(X), dev(Y)).cpu().numpy()
        assert np.array_equal(out, plain), f"pipe={pipe}"
        E = gen.features((g.nnz, 1), 1202, 1, gen.UNIT)
        with tuned(g.h, sddmm_pipe=pipe):
            em = fgp.sddmm(g.h, dev(X), dev(Y), E=dev(E)).cpu().numpy()
        assert np.array_equal(em.ravel(), (plain.ravel() * E.ravel()).astype(np.float32)), f"e_mul pipe={pipe}"
    for order, seg, rb in ((0, 1, 0), (1, 1, 1), (1, 1, 2), (1, 2, 1)):
        with tuned(g.h, sddmm_order=order, sddmm_seg_mb=seg, sddmm_rb_mb=rb, sddmm_seg_min_mb=0):
            g.h.prepare(F * 4)
            for pipe in (0, -1):
                with tuned(g.h, sddmm_pipe=pipe):
                    out = fgp.sddmm(g.h, dev(X), dev(Y)).cpu().numpy()
                assert np.array_equal(out, plain), f"order={order} seg={seg} rb={rb} pipe={pipe}"


@pytest.mark.parametrize("H,D", [(8, 32), (4, 64), (16, 32), (6, 32), (3, 64), (2, 64), (12, 32), (6, 64),
                                 (8, 64), (10, 32)])
@pytest.mark.parametrize("use_eid", [False, True])
def test_sddmm_heads_unit_prefetch(skewed, skewed_eid, H, D, use_eid):
    """a4: the unit-prefetching multi-head kernel (FG_TUNE_SDDMM_PIPE = 4, heads of
    D = 32 / 64) against the oracle, and bit for bit against the plain kernel
    (same lane partition and reduction tree), also with the e_mul write-back."""
    import paper_2008_11359_b200 as fgp
    g = skewed_eid if use_eid else skewed
    F = H * D
    X = feats((g.n_src, F), 1400 + F, gen.REAL)
    Y = feats((g.n_dst, F), 1401 + F, gen.REAL)
    ref, ab = oracle.sddmm(g.row_ptr, g.col_idx, X, Y, H=H)
    pos = np.arange(g.nnz) if g.eid is None else g.eid
    with tuned(g.h, sddmm_pipe=0):
        plain = fgp.sddmm(g.h, dev(X), dev(Y), H=H).cpu().numpy()
    E = gen.features((g.nnz, H), 1402, 1, gen.UNIT)
    for pipe in (4, 7, -1):
        with tuned(g.h, sddmm_pipe=pipe):
            out = fgp.sddmm(g.h, dev(X), dev(Y), H=H).cpu().numpy()
        check_close(out[pos], ref, ab, TOL, f"u_dot_v H={H} D={D} pf pipe={pipe}")
        assert np.array_equal(out, plain), f"pipe={pipe}"
        with tuned(g.h, sddmm_pipe=pipe):
            em = fgp.sddmm(g.h, dev(X), dev(Y), H=H, E=dev(E)).cpu().numpy()
        assert np.array_equal(em, (plain * E).astype(np.float32)), f"e_mul pipe={pipe}"
        with tuned(g.h, sddmm_seg_mb=1, sddmm_seg_min_mb=0):   # source-segmented unit tables
            g.h.prepare(F * 4)
            with tuned(g.h, sddmm_pipe=pipe):
                seg = fgp.sddmm(g.h, dev(X), dev(Y), H=H).cpu().numpy()
        assert np.array_equal(seg, plain), f"segmented pipe={pipe}"


@pytest.mark.parametrize("chunk", ["40", "128"])
def test_sddmm_unit_chunk_override(skewed, chunk, monkeypatch):
    """a4: work units of a non-default size (FG_SDDMM_CHUNK, read by
    fg_graph_create): 40 edges (not a multiple of a warp; the unit-prefetching
    kernels stage partial index batches) and 128 (above the prefetching kernels'
    64-edge buffers: those fall back to the plain kernel) -- H = 1 at F = 256 /
    512 and H = 8 D = 32, segmented and not, against the oracle."""
    import paper_2008_11359_b200 as fgp
    monkeypatch.setenv("FG_SDDMM_CHUNK", chunk)
    g = G(skewed.row_ptr, skewed.col_idx, skewed.n_src)
    for H, F in ((1, 256), (1, 512), (8, 256)):
        X = feats((g.n_src, F), 1500 + F + H, gen.REAL)
        Y = feats((g.n_dst, F), 1501 + F + H, gen.REAL)
        ref, ab = oracle.sddmm(g.row_ptr, g.col_idx, X, Y, H=H)
        out = fgp.sddmm(g.h, dev(X), dev(Y), H=H).cpu().numpy()
        check_close(out, ref, ab, TOL, f"u_dot_v H={H} F={F} chunk={chunk}")
        with tuned(g.h, sddmm_seg_mb=1, sddmm_seg_min_mb=0):
            g.h.prepare(F * 4)
            seg = fgp.sddmm(g.h, dev(X), dev(Y), H=H).cpu().numpy()
        check_close(seg, ref, ab, TOL, f"segmented u_dot_v H={H} F={F} chunk={chunk}")


@pytest.mark.parametrize("F", [8, 32, 40, 128, 512])
@pytest.mark.parametrize("red", ["sum", "max", "min", "mean"])
def test_copy_u_ldg256_pairs(skewed, F, red):
    """Ablation FG_TUNE_SPMM_LDG256: fp32 chunk pairs read with 32-byte loads,
    also under forced column tiling, against the oracle (max / min: values and
    argmax bit-exact)."""
    import paper_2008_11359_b200 as fgp
    g = skewed
    X = feats((g.n_src, F), 1300 + F, gen.REAL)
    ref, ab, rau, rae = oracle.spmm(g.row_ptr, g.col_idx, "copy_u", red, X)
    for tile_mb in (-1, 1):
        with tuned(g.h, spmm_ldg256=1, l2_tile_mb=tile_mb):
            if red in ("sum", "mean"):
                out = fgp.spmm(g.h, "copy_u", red, dev(X)).cpu().numpy()
                check_close(out, ref, ab, TOL, f"ldg256 copy_u-{red} F={F}")
            else:
                out, au, ae = fgp.spmm(g.h, "copy_u", red, dev(X), arg_u=True, arg_e=True)
                assert np.array_equal(out.cpu().numpy().astype(np.float64), ref)
                assert np.array_equal(au.cpu().numpy(), rau)
                assert np.array_equal(ae.cpu().numpy(), rae)


# ------------------------------------------------------------------ fused GAT (f2)
@pytest.mark.parametrize("H,D", [(8, 32), (4, 16), (2, 4), (1, 128), (8, 64), (1, 16), (16, 16), (4, 64), (2, 128),
                                 (6, 32), (4, 32), (8, 16), (2, 64), (3, 32), (16, 32), (4, 128)])
@pytest.mark.parametrize("use_eid", [False, True])
def test_gat_fused(skewed, skewed_eid, H, D, use_eid):
    import paper_2008_11359_b200 as fgp
    g = skewed_eid if use_eid else skewed
    X = feats((g.n_src, H * D), 970 + D, gen.REAL) * 0.5
    Y = feats((g.n_dst, H * D), 971 + D, gen.REAL) * 0.5
    out, sc = fgp.gat_attention(g.h, dev(X), dev(Y), H=H, scores=True)
    ref, ab = oracle.gat(g.row_ptr, g.col_idx, X, Y, H=H)
    check_close(out.cpu().numpy(), ref, ab, TOL, f"gat fused H={H} D={D}")
    rs, rab = oracle.sddmm(g.row_ptr, g.col_idx, X, Y, H=H)
    pos = np.arange(g.nnz) if g.eid is None else g.eid
    check_close(sc.cpu().numpy()[pos], rs, rab, TOL, "gat fused scores")
    # the unfused chain agrees with the fused op
    s = fgp.sddmm(g.h, dev(X), dev(Y), H=H)
    a = fgp.edge_softmax(g.h, s, H=H)
    o2 = fgp.spmm(g.h, "u_mul_e", "sum", dev(X), H=H, E=a).cpu().numpy()
    check_close(o2, ref, ab, TOL, "unfused chain")


@pytest.mark.parametrize("H,D", [(3, 12), (4, 3), (2, 6), (16, 64), (6, 20), (3, 44)])
@pytest.mark.parametrize("use_eid", [False, True])
def test_sddmm_generic_heads(skewed, skewed_eid, H, D, use_eid):
    """Head shapes outside the lane-partitioned kernels (D not 4 * 2^k, or
    H*D > 512): the generic thread-per-edge kernel, plain, segmented and with
    the e_mul scale, against the oracle."""
    import paper_2008_11359_b200 as fgp
    g = skewed_eid if use_eid else skewed
    X = feats((g.n_src, H * D), 1400 + D, gen.REAL)
    Y = feats((g.n_dst, H * D), 1401 + D, gen.REAL)
    ref, ab = oracle.sddmm(g.row_ptr, g.col_idx, X, Y, H=H)
    pos = np.arange(g.nnz) if g.eid is None else g.eid
    out = fgp.sddmm(g.h, dev(X), dev(Y), H=H).cpu().numpy()
    check_close(out[pos], ref, ab, TOL, f"generic u_dot_v H={H} D={D}")
    with tuned(g.h, sddmm_seg_mb=1, sddmm_seg_min_mb=0):
        g.h.prepare(H * D * 4)
        seg = fgp.sddmm(g.h, dev(X), dev(Y), H=H).cpu().numpy()
    assert np.array_equal(seg, out)               # same per-edge arithmetic, other unit order
    E = gen.features((g.nnz, H), 1402, 1, gen.UNIT)
    em = fgp.sddmm(g.h, dev(X), dev(Y), H=H, E=dev(E)).cpu().numpy()
    assert np.array_equal(em, (out * E).astype(np.float32))


@pytest.mark.parametrize("H,D", [(3, 12), (4, 3), (16, 64), (1, 256), (2, 6)])
def test_gat_unfused_fallback(skewed, H, D):
    """fg_gat_attention outside the fused kernel's shapes: the unfused chain
    through the scores buffer (include/fg.h), against the GAT definition; the
    scores buffer ends with the pre-softmax scores; without it FG_EUNSUPPORTED."""
    import paper_2008_11359_b200 as fgp
    g = skewed
    X = feats((g.n_src, H * D), 1410 + D, gen.REAL) * 0.5
    Y = feats((g.n_dst, H * D), 1411 + D, gen.REAL) * 0.5
    out, sc = fgp.gat_attention(g.h, dev(X), dev(Y), H=H, scores=True)
    ref, ab = oracle.gat(g.row_ptr, g.col_idx, X, Y, H=H)
    check_close(out.cpu().numpy(), ref, ab, TOL, f"gat fallback H={H} D={D}")
    rs, rab = oracle.sddmm(g.row_ptr, g.col_idx, X, Y, H=H)
    check_close(sc.cpu().numpy(), rs, rab, TOL, "gat fallback scores")
    with pytest.raises(fgp.FGError) as e:
        fgp.gat_attention(g.h, dev(X), dev(Y), H=H)
    assert e.value.status == 3   # FG_EUNSUPPORTED


# ------------------------------------------------------------------ bf16 feature storage (row f4)
def bf16_dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).cuda().view(torch.bfloat16)


@pytest.mark.parametrize("F", [4, 32, 128, 200, 512, 640])
@pytest.mark.parametrize("red", ["sum", "max", "min", "mean"])
def test_copy_u_bf16(skewed, F, red):
    """fg_spmm_x16: the oracle runs on the exact fp32 decoding of the same bf16
    inputs; sum to tolerance, max values and argmax exact."""
    import paper_2008_11359_b200 as fgp
    bits, dec = gen.to_bf16(feats((skewed.n_src, F), 700 + F, gen.REAL))
    ref, ab, rau, rae = oracle.spmm(skewed.row_ptr, skewed.col_idx, "copy_u", red, dec)
    if red in ("sum", "mean"):
        out = fgp.spmm(skewed.h, "copy_u", red, bf16_dev(bits)).cpu().numpy()
        check_close(out, ref, ab, TOL, f"bf16 copy_u-{red} F={F}")
    else:
        out, au, ae = fgp.spmm(skewed.h, "copy_u", red, bf16_dev(bits), arg_u=True, arg_e=True)
        assert np.array_equal(out.cpu().numpy().astype(np.float64), ref)
        assert np.array_equal(au.cpu().numpy(), rau) and np.array_equal(ae.cpu().numpy(), rae)


@pytest.mark.parametrize("H,D", [(8, 32), (4, 2), (1, 512)])
@pytest.mark.parametrize("red", ["sum", "max", "min", "mean"])
@pytest.mark.parametrize("use_eid", [False, True])
def test_u_mul_e_bf16(skewed, skewed_eid, H, D, red, use_eid):
    import paper_2008_11359_b200 as fgp
    g = skewed_eid if use_eid else skewed
    bits, dec = gen.to_bf16(feats((g.n_src, H * D), 710 + D, gen.REAL))
    E = gen.features((g.nnz, H), 711, 0, gen.UNIT)
    ref, ab, rau, rae = oracle.spmm(g.row_ptr, g.col_idx, "u_mul_e", red, dec, H=H, E=E, eid=g.eid)
    if red in ("sum", "mean"):
        out = fgp.spmm(g.h, "u_mul_e", red, bf16_dev(bits), H=H, E=dev(E)).cpu().numpy()
        check_close(out, ref, ab, TOL, f"bf16 u_mul_e-{red} H={H} D={D}")
    else:
        out, au, ae = fgp.spmm(g.h, "u_mul_e", red, bf16_dev(bits), H=H, E=dev(E), arg_u=True, arg_e=True)
        assert np.array_equal(out.cpu().numpy().astype(np.float64), ref)
        assert np.array_equal(au.cpu().numpy(), rau) and np.array_equal(ae.cpu().numpy(), rae)


@pytest.mark.parametrize("H,D", [(1, 16), (1, 128), (1, 512), (8, 32), (2, 4), (4, 64), (2, 16), (16, 8), (4, 128), (2, 256)])
@pytest.mark.parametrize("use_eid", [False, True])
def test_sddmm_bf16(skewed, skewed_eid, H, D, use_eid):
    import paper_2008_11359_b200 as fgp
    g = skewed_eid if use_eid else skewed
    xb, xd = gen.to_bf16(feats((g.n_src, H * D), 720 + D, gen.REAL))
    yb, yd = gen.to_bf16(feats((g.n_dst, H * D), 721 + D, gen.REAL))
    out = fgp.sddmm(g.h, bf16_dev(xb), bf16_dev(yb), H=H).cpu().numpy()
    ref, ab = oracle.sddmm(g.row_ptr, g.col_idx, xd, yd, H=H)
    pos = np.arange(g.nnz) if g.eid is None else g.eid
    check_close(out[pos], ref, ab, TOL, f"bf16 u_dot_v H={H} D={D}")


def test_bf16_rejects_unsupported(skewed):
    import paper_2008_11359_b200 as fgp
    bits, _ = gen.to_bf16(feats((skewed.n_src, 32), 730, gen.REAL))
    E = torch.zeros(skewed.nnz, 1, device="cuda")
    with pytest.raises(fgp.FGError) as e:
        fgp.spmm(skewed.h, "u_add_e", "sum", bf16_dev(bits), E=E)
    assert e.value.status == 3   # FG_EUNSUPPORTED


@pytest.mark.parametrize("F", [128, 512])
def test_copy_u_bf16_tiled_and_unaligned(skewed, F):
    """bf16 storage on the column-tiled copy_u path (a 1 MiB L2 budget forces
    tiles on this graph) and with an X that is 8- but not 16-byte aligned (the
    8-byte-per-chunk mapping instead of 16-byte pair loads)."""
    import paper_2008_11359_b200 as fgp
    bits, dec = gen.to_bf16(feats((skewed.n_src, F), 740 + F, gen.REAL))
    ref, ab, _, _ = oracle.spmm(skewed.row_ptr, skewed.col_idx, "copy_u", "sum", dec)
    with tuned(skewed.h, l2_tile_mb=1):
        out = fgp.spmm(skewed.h, "copy_u", "sum", bf16_dev(bits)).cpu().numpy()
    check_close(out, ref, ab, TOL, f"bf16 copy_u-sum tiled F={F}")
    buf = torch.empty(skewed.n_src * F + 4, dtype=torch.bfloat16, device="cuda")
    Xu = buf[4:].view(skewed.n_src, F)            # 8-byte aligned, not 16
    Xu.copy_(bf16_dev(bits))
    out = fgp.spmm(skewed.h, "copy_u", "sum", Xu).cpu().numpy()
    check_close(out, ref, ab, TOL, f"bf16 copy_u-sum unaligned F={F}")
    Yb, Yd = gen.to_bf16(feats((skewed.n_dst, F), 741 + F, gen.REAL))
    s = fgp.sddmm(skewed.h, Xu, bf16_dev(Yb), H=1).cpu().numpy()
    rs, rab = oracle.sddmm(skewed.row_ptr, skewed.col_idx, dec, Yd, H=1)
    check_close(s, rs, rab, TOL, f"bf16 u_dot_v unaligned F={F}")


# ------------------------------------------------------------------ u_dot_v then e_mul (row f4)
@pytest.mark.parametrize("H,D", [(1, 512), (1, 16), (8, 32), (2, 4), (64, 4)])
@pytest.mark.parametrize("use_eid", [False, True])
def test_sddmm_emul(skewed, skewed_eid, H, D, use_eid):
    """fg_sddmm_emul vs the oracle (score * E[eid][h]); (64, 4) has more heads than
    a group stages, so the scale runs as a second pass."""
    import paper_2008_11359_b200 as fgp
    g = skewed_eid if use_eid else skewed
    X = feats((g.n_src, H * D), 990 + D, gen.REAL)
    Y = feats((g.n_dst, H * D), 991 + D, gen.REAL)
    E = gen.features((g.nnz, H), 992, 0, gen.REAL) * np.float32(3)
    out = fgp.sddmm(g.h, dev(X), dev(Y), H=H, E=dev(E)).cpu().numpy()
    ref, ab = oracle.sddmm_emul(g.row_ptr, g.col_idx, X, Y, E, H=H, eid=g.eid)
    pos = np.arange(g.nnz) if g.eid is None else g.eid
    check_close(out[pos], ref, ab, TOL, f"u_dot_v-e_mul H={H} D={D}")
    # integer regime: exact
    Xi, Yi = feats((g.n_src, H * D), 993, gen.INT), feats((g.n_dst, H * D), 994, gen.INT)
    Ei = gen.features((g.nnz, H), 995, 0, gen.INT, lo=-3, hi=3)
    out = fgp.sddmm(g.h, dev(Xi), dev(Yi), H=H, E=dev(Ei)).cpu().numpy()
    ref, _ = oracle.sddmm_emul(g.row_ptr, g.col_idx, Xi, Yi, Ei, H=H, eid=g.eid)
    assert np.array_equal(out[pos].astype(np.float64), ref)


def test_sddmm_emul_rejects_overlap(skewed):
    import paper_2008_11359_b200 as fgp
    X = dev(feats((skewed.n_src, 32), 996, gen.REAL))
    E = dev(gen.features((skewed.nnz, 1), 997, 0, gen.REAL))
    with pytest.raises(fgp.FGError) as e:
        fgp.sddmm(skewed.h, X, H=1, E=E, out=E)
    assert e.value.status == 1   # FG_EINVAL


# ------------------------------------------------------------------ bipartite (n_src != n_dst)
@pytest.fixture(scope="module")
def bipartite():
    """1,500 destinations over 4,000 sources, 90K edges, lognormal in-degrees up to
    3,500 (CTA-per-row rows), uniform sources, 20 empty rows."""
    deg = gen.degrees_lognormal(1500, 90000, 1.4, 3500, 61)
    deg[gen.permutation(1500, 62)[:20]] = 0
    g = gen.csr_from_degrees(deg, 4000, 63, uniform_sources=True)
    return G(g.row_ptr, g.col_idx, n_src=4000)


def test_bipartite_all_ops(bipartite):
    import paper_2008_11359_b200 as fgp
    g = bipartite
    for F in (32, 512):
        X = feats((g.n_src, F), 1100 + F, gen.REAL)
        out = fgp.spmm(g.h, "copy_u", "sum", dev(X)).cpu().numpy()
        ref, ab, _, _ = oracle.spmm(g.row_ptr, g.col_idx, "copy_u", "sum", X)
        check_close(out, ref, ab, TOL, f"bipartite copy_u-sum F={F}")
        o, au, ae = fgp.spmm(g.h, "copy_u", "max", dev(X), arg_u=True, arg_e=True)
        ref, _, rau, rae = oracle.spmm(g.row_ptr, g.col_idx, "copy_u", "max", X)
        assert np.array_equal(o.cpu().numpy().astype(np.float64), ref)
        assert np.array_equal(au.cpu().numpy(), rau) and np.array_equal(ae.cpu().numpy(), rae)
        bits, dec = gen.to_bf16(X)
        ob = fgp.spmm(g.h, "copy_u", "sum", bf16_dev(bits)).cpu().numpy()
        ref, ab, _, _ = oracle.spmm(g.row_ptr, g.col_idx, "copy_u", "sum", dec)
        check_close(ob, ref, ab, TOL, f"bipartite bf16 copy_u-sum F={F}")
    H, D = 8, 32
    X = feats((g.n_src, H * D), 1110, gen.REAL)
    Y = feats((g.n_dst, H * D), 1111, gen.REAL)
    s = fgp.sddmm(g.h, dev(X), dev(Y), H=H)
    rs, rab = oracle.sddmm(g.row_ptr, g.col_idx, X, Y, H=H)
    check_close(s.cpu().numpy(), rs, rab, TOL, "bipartite u_dot_v H=8")
    rs32 = rs.astype(np.float32)
    a = fgp.edge_softmax(g.h, dev(rs32), H=H).cpu().numpy().astype(np.float64)
    ra = oracle.edge_softmax(g.row_ptr, rs32, H=H)
    assert (np.abs(a - ra) <= TOL * ra).all()
    ra32 = ra.astype(np.float32)
    o = fgp.spmm(g.h, "u_mul_e", "sum", dev(X), H=H, E=dev(ra32)).cpu().numpy()
    ro, rob, _, _ = oracle.spmm(g.row_ptr, g.col_idx, "u_mul_e", "sum", X, H=H, E=ra32)
    check_close(o, ro, rob, TOL, "bipartite u_mul_e-sum H=8")
    X8 = feats((g.n_src, 8), 1112, gen.INT)
    Xd = feats((g.n_dst, 8), 1113, gen.INT)
    W = gen.features((8, 128), 1114, 1, gen.INT, lo=-4, hi=4)
    om, amu, ame = fgp.spmm(g.h, "mlp", "max", dev(X8), W=dev(W), X_dst=dev(Xd), arg_u=True, arg_e=True)
    rm, _, rmu, rme = oracle.spmm(g.row_ptr, g.col_idx, "mlp", "max", X8, W=W, X_dst=Xd)
    assert np.array_equal(om.cpu().numpy().astype(np.float64), rm)
    assert np.array_equal(amu.cpu().numpy(), rmu) and np.array_equal(ame.cpu().numpy(), rme)
    gat = fgp.gat_attention(g.h, dev(X), dev(Y), H=H).cpu().numpy()
    rg, rgb = oracle.gat(g.row_ptr, g.col_idx, X, Y, H=H)
    check_close(gat, rg, rgb, TOL, "bipartite fused GAT")


@pytest.mark.parametrize("chunk", ["32", "256"])
def test_sddmm_unit_sizes(skewed, monkeypatch, chunk):
    """The SDDMM work-unit size (edges per unit, fixed at graph creation;
    default 64) does not change any result: same per-edge arithmetic."""
    import paper_2008_11359_b200 as fgp
    monkeypatch.setenv("FG_SDDMM_CHUNK", chunk)
    g2 = G(skewed.row_ptr, skewed.col_idx, skewed.n_src)
    for H, D in ((1, 512), (8, 32)):
        X = feats((skewed.n_src, H * D), 1200 + D, gen.REAL)
        a = fgp.sddmm(g2.h, dev(X), H=H).cpu().numpy()
        b = fgp.sddmm(skewed.h, dev(X), H=H).cpu().numpy()
        assert np.array_equal(a, b)


# ------------------------------------------------------------------ CTA-per-row path on the small graphs
@pytest.mark.parametrize("deg", ["1", "200", "1024"])
def test_cta_per_row_thresholds(skewed, skewed_eid, deg):
    """Rows of degree >= FG_SPMM_HEAVY_DEG / FG_GAT_HEAVY_DEG (default 4096, above
    this graph's maximum) run CTA-per-row with the fixed-order combine: force it
    for most rows and check sum / max (argmax ties across the CTA's chunks) / min /
    mean, u_mul_e and u_add_e with edge ids, bf16 storage and the fused GAT."""
    d = int(deg)
    with tuned(skewed.h, spmm_heavy_deg=d, gat_heavy_deg=d), tuned(skewed_eid.h, spmm_heavy_deg=d, gat_heavy_deg=d):
        _cta_per_row_thresholds(skewed, skewed_eid)


def _cta_per_row_thresholds(skewed, skewed_eid):
    import paper_2008_11359_b200 as fgp
    g = skewed
    for F, regime in ((512, gen.REAL), (32, gen.INT), (128, gen.INT)):
        X = feats((g.n_src, F), 1300 + F, regime, lo=-2, hi=2)   # integers in [-2, 2]: many ties
        for red in ("sum", "max", "min", "mean"):
            ref, ab, rau, rae = oracle.spmm(g.row_ptr, g.col_idx, "copy_u", red, X)
            if red in ("max", "min"):
                o, au, ae = fgp.spmm(g.h, "copy_u", red, dev(X), arg_u=True, arg_e=True)
                assert np.array_equal(o.cpu().numpy().astype(np.float64), ref), (red, F)
                assert np.array_equal(au.cpu().numpy(), rau) and np.array_equal(ae.cpu().numpy(), rae), (red, F)
            else:
                check_close(fgp.spmm(g.h, "copy_u", red, dev(X)).cpu().numpy(), ref, ab, TOL, f"{red} F={F}")
    ge = skewed_eid
    H, D = 8, 32
    X = feats((ge.n_src, H * D), 1310, gen.REAL)
    E = gen.features((ge.nnz, H), 1311, 0, gen.UNIT)
    for op in ("u_mul_e", "u_add_e"):
        ref, ab, _, _ = oracle.spmm(ge.row_ptr, ge.col_idx, op, "sum", X, H=H, E=E, eid=ge.eid)
        check_close(fgp.spmm(ge.h, op, "sum", dev(X), H=H, E=dev(E)).cpu().numpy(), ref, ab, TOL, op)
    bits, dec = gen.to_bf16(X)
    ref, ab, _, _ = oracle.spmm(g.row_ptr, g.col_idx, "copy_u", "sum", dec)
    check_close(fgp.spmm(g.h, "copy_u", "sum", bf16_dev(bits)).cpu().numpy(), ref, ab, TOL, "bf16 copy_u")
    Y = feats((g.n_dst, H * D), 1312, gen.REAL)
    out = fgp.gat_attention(g.h, dev(X), dev(Y), H=H).cpu().numpy()
    rg, rgb = oracle.gat(g.row_ptr, g.col_idx, X, Y, H=H)
    check_close(out, rg, rgb, TOL, "fused GAT")


# ------------------------------------------------------------------ randomized equivalence
def test_random_equivalence_200_cases():
    """200 seeded random cases -- graph size and skew, feature shape, message,
    reducer, edge-id permutation, regime -- each GPU op against the oracle, with
    every output pre-filled with NaN / garbage (outputs must be fully overwritten)."""
    import paper_2008_11359_b200 as fgp
    rng = np.random.default_rng(20081135)
    shapes = [(1, 4), (1, 12), (1, 32), (1, 100), (1, 512), (2, 4), (4, 8), (8, 32), (2, 64), (3, 12)]
    for case in range(200):
        n = int(rng.integers(1, 400))
        n_src = n if rng.random() < 0.7 else int(rng.integers(1, 500))
        m = int(rng.integers(0, min(n * n_src, 6000) + 1))
        deg = rng.multinomial(m, rng.dirichlet(np.full(n, float(rng.choice([0.2, 1.0, 5.0]))))) if m else np.zeros(n, int)
        deg = np.minimum(deg, n_src)
        rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
        ci = np.concatenate([np.sort(rng.choice(n_src, size=int(d), replace=False)) for d in deg]
                            + [np.zeros(0, np.int64)]).astype(np.int32)
        eid = rng.permutation(int(rp[-1])).astype(np.int32) if rng.random() < 0.3 else None
        g = G(rp, ci, n_src=n_src, eid=eid)
        H, D = shapes[int(rng.integers(len(shapes)))]
        F = H * D
        regime = gen.INT if rng.random() < 0.3 else gen.REAL
        X = feats((n_src, F), 5000 + case, regime)
        what = f"case {case}: n={n} n_src={n_src} m={g.nnz} H={H} D={D} eid={eid is not None}"
        kind = case % 4
        if kind == 0:   # copy_u / u_mul_e with a random reducer
            msg = "copy_u" if rng.random() < 0.5 else "u_mul_e"
            red = str(rng.choice(["sum", "max", "min", "mean"]))
            E = gen.features((max(g.nnz, 1), H), 6000 + case, 0, gen.UNIT)[: g.nnz] if msg == "u_mul_e" else None
            out = torch.full((n, F), float("nan"), device="cuda")
            kw = dict(H=H, out=out)
            if E is not None:
                kw["E"] = dev(E) if g.nnz else torch.zeros((0, H), device="cuda")
            if red in ("max", "min"):
                au = torch.full((n, F), 12345, dtype=torch.int32, device="cuda")
                fgp.spmm(g.h, msg, red, dev(X), arg_u=au, **kw)
            else:
                fgp.spmm(g.h, msg, red, dev(X), **kw)
            ref, ab, rau, _ = oracle.spmm(g.row_ptr, g.col_idx, msg, red, X, H=H, E=E, eid=g.eid)
            if red in ("max", "min"):
                assert np.array_equal(out.cpu().numpy().astype(np.float64), ref), what
                assert np.array_equal(au.cpu().numpy(), rau), what
            else:
                check_close(out.cpu().numpy(), ref, ab, TOL, what)
        elif kind == 1:   # u_dot_v
            if D % 4 or (H > 1 and (D // 4) & (D // 4 - 1)):
                H, D = 1, F
            Y = feats((n, F), 7000 + case, regime)
            out = torch.full((max(g.nnz, 1), H), float("nan"), device="cuda")[: g.nnz]
            fgp.sddmm(g.h, dev(X), dev(Y), H=H, out=out)
            ref, ab = oracle.sddmm(g.row_ptr, g.col_idx, X, Y, H=H)
            pos = np.arange(g.nnz) if g.eid is None else g.eid
            check_close(out.cpu().numpy()[pos], ref, ab, TOL, what)
        elif kind == 2:   # edge softmax on oracle scores
            S = gen.features((max(g.nnz, 1), H), 8000 + case, 0, gen.REAL)[: g.nnz] * np.float32(6)
            if g.nnz == 0:
                continue
            out = torch.full((g.nnz, H), float("nan"), device="cuda")
            fgp.edge_softmax(g.h, dev(S), H=H, out=out)
            ref = oracle.edge_softmax(g.row_ptr, S, H=H, eid=g.eid)
            pos = np.arange(g.nnz) if g.eid is None else g.eid
            got = out.cpu().numpy()[pos].astype(np.float64)
            assert (np.abs(got - ref) <= TOL * ref).all(), what
        else:   # mlp max / sum (integer regime: exact)
            d2 = int(rng.choice([16, 32, 128, 200]))
            X8 = feats((n_src, 8), 9000 + case, gen.INT)
            Xd = feats((n, 8), 9100 + case, gen.INT)
            W = gen.features((8, d2), 9200 + case, 1, gen.INT, lo=-4, hi=4)
            red = "max" if rng.random() < 0.6 else "sum"
            out = torch.full((n, d2), float("nan"), device="cuda")
            if red == "max":
                au = torch.full((n, d2), 12345, dtype=torch.int32, device="cuda")
                fgp.spmm(g.h, "mlp", "max", dev(X8), W=dev(W), X_dst=dev(Xd), out=out, arg_u=au)
            else:
                fgp.spmm(g.h, "mlp", "sum", dev(X8), W=dev(W), X_dst=dev(Xd), out=out)
            ref, _, rau, _ = oracle.spmm(g.row_ptr, g.col_idx, "mlp", red, X8, W=W, X_dst=Xd, eid=g.eid)
            assert np.array_equal(out.cpu().numpy().astype(np.float64), ref), what
            if red == "max":
                assert np.array_equal(au.cpu().numpy(), rau), what
