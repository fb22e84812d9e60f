"""Pins for the fp64 oracle against things other than itself (CPU only).

Each check is chosen so a plausible mistake in oracle/oracle.c (dropped term,
wrong sign/index, transposed operand, wrong tie rule, wrong edge direction)
fails at least one of them:
  * dense A.X (Eq. (3)) and |A|.|X| for the abs-sums;
  * all-ones X -> in-degree exactly;
  * numpy masked max / first-occurrence argmax; relabelling invariance;
  * weighted dense A_w.X per head, E == 1 reduces to copy_u;
  * MLP max closed form ReLU(max_u (XW)[u] + (XW)[v]) (distributivity +
    monotone ReLU), brute-force MLP sum;
  * complete graph u_dot_v == dense X.Y^T per head (Eq. (4));
  * adjoint identity of the gradient duality;
  * softmax: rows sum to 1, shift invariance, constant -> 1/deg, torch.softmax
    on a dense -inf-masked matrix;
  * SPEC.md worked examples in tests/golden/spec_examples.json;
  * row f4: numpy masked min / argmin, min = -max(-.), mean = dense A_w.X / deg,
    u_add_e = A.X + A_E.1, masked max/min of fp32 x_u + e, copy_e = row sums /
    masked max of the E-weighted adjacency, u_OP_v on the complete graph = the
    dense broadcast, sum_j u_mul_v = u_dot_v.
"""
import json
import os

import numpy as np
import pytest

import gen
import oracle
from helpers import csr_from_edges, dense_adjacency, edge_rows

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def small_graph(n=257, m=3000, seed=5, empty_rows=True, uniform=False):
    g = gen.random_graph(n, m, seed, sigma=1.0, n_empty=max(1, n // 20) if empty_rows else 0,
                         uniform_sources=uniform)
    assert (g.degrees() == 0).any() == empty_rows
    return g


# ------------------------------------------------------------------ copy_u
@pytest.mark.parametrize("F", [1, 4, 12, 32])
def test_copy_u_sum_dense(F):
    g = small_graph()
    X = gen.features((g.n_src, F), 11, 0)
    ref, ab, _, _ = oracle.spmm(g.row_ptr, g.col_idx, "copy_u", "sum", X)
    A = dense_adjacency(g.row_ptr, g.col_idx, g.n_src)
    np.testing.assert_allclose(ref, A @ X.astype(np.float64), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(ab, A @ np.abs(X.astype(np.float64)), rtol=1e-12, atol=1e-12)


def test_copy_u_sum_ones_is_indegree():
    g = small_graph(n=500, m=9000)
    X = np.ones((g.n_src, 8), np.float32)
    ref, _, _, _ = oracle.spmm(g.row_ptr, g.col_idx, "copy_u", "sum", X)
    assert np.array_equal(ref, np.repeat(g.degrees()[:, None].astype(np.float64), 8, 1))


def test_spec_copy_u_example():
    ex = GOLD["copy_u_sum"]
    rp, ci = csr_from_edges(ex["n"], ex["edges"])
    ref, _, _, _ = oracle.spmm(rp, ci, "copy_u", "sum", np.array(ex["X"], np.float32))
    assert np.array_equal(ref, np.array(ex["expected"], np.float64))


def _masked_max(row_ptr, col_idx, n_src, M):
    """numpy masked max over messages M[v, u, j] (only edges u->v count),
    argmax = first occurrence along ascending u (== lowest CSR position)."""
    A = dense_adjacency(row_ptr, col_idx, n_src) > 0
    Mm = np.where(A[:, :, None], M, -np.inf)
    val = Mm.max(axis=1)
    arg = Mm.argmax(axis=1)
    empty = ~A.any(axis=1)
    val[empty] = 0.0
    arg[empty] = -1
    return val, arg


def _eid_of(row_ptr, col_idx, v, u):
    p = np.searchsorted(col_idx[row_ptr[v]:row_ptr[v + 1]], u) + row_ptr[v]
    assert col_idx[p] == u
    return p


@pytest.mark.parametrize("regime", [gen.REAL, gen.INT])
def test_copy_u_max_masked(regime):
    g = small_graph()
    X = gen.features((g.n_src, 6), 13, 0, regime, lo=-3, hi=3)   # INT: many ties
    ref, ab, au, ae = oracle.spmm(g.row_ptr, g.col_idx, "copy_u", "max", X)
    M = np.broadcast_to(X.astype(np.float64)[None], (g.n_dst, g.n_src, 6))
    val, arg = _masked_max(g.row_ptr, g.col_idx, g.n_src, M)
    assert np.array_equal(ref, val)
    assert np.array_equal(au, arg)
    assert np.array_equal(ab, np.abs(val))
    for v in range(0, g.n_dst, 7):
        for j in range(6):
            if arg[v, j] >= 0:
                assert ae[v, j] == _eid_of(g.row_ptr, g.col_idx, v, arg[v, j])
            else:
                assert ae[v, j] == -1


def test_copy_u_max_relabel_invariance():
    g = small_graph(n=120, m=1500, seed=9)
    X = gen.features((g.n_src, 5), 3, 0, gen.INT, lo=-4, hi=4)
    ref, _, au, _ = oracle.spmm(g.row_ptr, g.col_idx, "copy_u", "max", X)
    pi = gen.permutation(g.n_dst, 99)                 # new id of old vertex i = pi[i]
    src, dst = g.col_idx.astype(np.int64), edge_rows(g.row_ptr)
    rp2, ci2 = csr_from_edges(g.n_dst, np.stack([pi[src], pi[dst]], 1))
    X2 = np.empty_like(X)
    X2[pi] = X
    ref2, _, au2, _ = oracle.spmm(rp2, ci2, "copy_u", "max", X2)
    assert np.array_equal(ref2[pi], ref)
    # the max VALUE is relabelling-invariant; the winner is the same vertex when
    # no tie occurs (ties resolve by position, which relabelling changes)
    Xd = X.astype(np.float64)
    for v in range(g.n_dst):
        for j in range(5):
            if au[v, j] >= 0:
                assert Xd[au[v, j], j] == ref[v, j]
                assert X2[au2[pi[v], j], j] == ref[v, j]


@pytest.mark.parametrize("regime", [gen.REAL, gen.INT])
def test_copy_u_min_masked(regime):
    """min (row f4): numpy masked min with first-occurrence argmin."""
    g = small_graph()
    X = gen.features((g.n_src, 6), 14, 0, regime, lo=-3, hi=3)
    ref, ab, au, ae = oracle.spmm(g.row_ptr, g.col_idx, "copy_u", "min", X)
    A = dense_adjacency(g.row_ptr, g.col_idx, g.n_src) > 0
    Mm = np.where(A[:, :, None], X.astype(np.float64)[None], np.inf)
    val, arg = Mm.min(axis=1), Mm.argmin(axis=1)
    empty = ~A.any(axis=1)
    val[empty], arg[empty] = 0.0, -1
    assert np.array_equal(ref, val)
    assert np.array_equal(au, arg)
    assert np.array_equal(ab, np.abs(val))
    for v in range(0, g.n_dst, 5):
        for j in range(6):
            assert ae[v, j] == (_eid_of(g.row_ptr, g.col_idx, v, arg[v, j]) if arg[v, j] >= 0 else -1)


def test_u_mul_e_min_is_negated_max():
    """min_u t = -max_u (-t) with the same first-wins winner (negating E negates
    every fp32 product exactly)."""
    g = small_graph(n=150, m=2500, seed=12)
    H, D = 2, 4
    X = gen.features((g.n_src, H * D), 31, 0, gen.INT, lo=-3, hi=3)
    E = gen.features((g.nnz, H), 31, 1, gen.INT, lo=-2, hi=2)
    mn, _, au, ae = oracle.spmm(g.row_ptr, g.col_idx, "u_mul_e", "min", X, H=H, E=E)
    mx, _, au2, ae2 = oracle.spmm(g.row_ptr, g.col_idx, "u_mul_e", "max", X, H=H, E=-E)
    assert np.array_equal(mn, -mx + 0.0)
    assert np.array_equal(au, au2) and np.array_equal(ae, ae2)


@pytest.mark.parametrize("op", ["copy_u", "u_mul_e"])
def test_mean_is_dense_over_degree(op):
    """mean (row f4): (A_w X) / deg(v), empty rows 0."""
    g = small_graph()
    H, D = 2, 3
    X = gen.features((g.n_src, H * D), 17, 0)
    E = gen.features((g.nnz, H), 17, 1, gen.UNIT) if op == "u_mul_e" else None
    ref, ab, au, _ = oracle.spmm(g.row_ptr, g.col_idx, op, "mean", X, H=H, E=E)
    assert au is None
    deg = np.maximum(g.degrees(), 1).astype(np.float64)[:, None]
    for h in range(H):
        w = E[:, h].astype(np.float64) if E is not None else None
        Aw = dense_adjacency(g.row_ptr, g.col_idx, g.n_src, w)
        blk = slice(h * D, (h + 1) * D)
        np.testing.assert_allclose(ref[:, blk], Aw @ X[:, blk].astype(np.float64) / deg, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(ab[:, blk], np.abs(Aw) @ np.abs(X[:, blk].astype(np.float64)) / deg,
                                   rtol=1e-12, atol=1e-12)
    assert np.all(ref[g.degrees() == 0] == 0.0)


# ------------------------------------------------------------------ u_add_e, copy_e (row f4)
def test_u_add_e_sum_dense():
    """sum_p (x_u + e_p) = (A X)[v] + (A_E 1)[v] per head."""
    g = small_graph()
    H, D = 3, 4
    X = gen.features((g.n_src, H * D), 41, 0)
    E = gen.features((g.nnz, H), 41, 1)
    ref, ab, _, _ = oracle.spmm(g.row_ptr, g.col_idx, "u_add_e", "sum", X, H=H, E=E)
    A = dense_adjacency(g.row_ptr, g.col_idx, g.n_src)
    for h in range(H):
        Aw = dense_adjacency(g.row_ptr, g.col_idx, g.n_src, E[:, h].astype(np.float64))
        blk = slice(h * D, (h + 1) * D)
        want = A @ X[:, blk].astype(np.float64) + Aw.sum(axis=1)[:, None]
        np.testing.assert_allclose(ref[:, blk], want, rtol=1e-12, atol=1e-12)
        wabs = A @ np.abs(X[:, blk].astype(np.float64)) + np.abs(Aw).sum(axis=1)[:, None]
        np.testing.assert_allclose(ab[:, blk], wabs, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("red", ["max", "min"])
def test_u_add_e_select_masked(red):
    """max/min over fp32-rounded x_u + e_p (numpy fp32 add is IEEE RN), first wins."""
    g = small_graph(n=180, m=2600, seed=21)
    H, D = 2, 2
    X = gen.features((g.n_src, H * D), 43, 0, gen.INT, lo=-3, hi=3)
    E = gen.features((g.nnz, H), 43, 1, gen.INT, lo=-2, hi=2)
    ref, _, au, ae = oracle.spmm(g.row_ptr, g.col_idx, "u_add_e", red, X, H=H, E=E)
    A = dense_adjacency(g.row_ptr, g.col_idx, g.n_src) > 0
    rows = edge_rows(g.row_ptr)
    Ed = np.zeros((g.n_dst, g.n_src, H), np.float32)
    Ed[rows, g.col_idx] = E
    M = (X[None, :, :] + np.repeat(Ed, D, axis=2)).astype(np.float64)
    fill = -np.inf if red == "max" else np.inf
    Mm = np.where(A[:, :, None], M, fill)
    val = Mm.max(axis=1) if red == "max" else Mm.min(axis=1)
    arg = Mm.argmax(axis=1) if red == "max" else Mm.argmin(axis=1)
    empty = ~A.any(axis=1)
    val[empty], arg[empty] = 0.0, -1
    assert np.array_equal(ref, val)
    assert np.array_equal(au, arg)


@pytest.mark.parametrize("red", ["sum", "max"])
def test_copy_e_dense(red):
    """copy_e: the message is the edge's own row; sum = row sums of the E-weighted
    adjacency, max = masked max over it (first occurrence)."""
    g = small_graph()
    F = 5
    E = gen.features((g.nnz, F), 45, 0, gen.INT if red == "max" else gen.REAL, lo=-3, hi=3)
    eid = gen.permutation(g.nnz, 46).astype(np.int32)
    ref, ab, au, ae = oracle.spmm(g.row_ptr, g.col_idx, "copy_e", red, None, E=E, eid=eid)
    A = dense_adjacency(g.row_ptr, g.col_idx, g.n_src) > 0
    for j in range(F):
        Aw = dense_adjacency(g.row_ptr, g.col_idx, g.n_src, E[eid, j].astype(np.float64))   # value at CSR pos
        if red == "sum":
            np.testing.assert_allclose(ref[:, j], Aw.sum(axis=1), rtol=1e-12, atol=1e-12)
            np.testing.assert_allclose(ab[:, j], np.abs(Aw).sum(axis=1), rtol=1e-12, atol=1e-12)
        else:
            Mm = np.where(A, Aw, -np.inf)
            val, arg = Mm.max(axis=1), Mm.argmax(axis=1)
            empty = ~A.any(axis=1)
            val[empty], arg[empty] = 0.0, -1
            assert np.array_equal(ref[:, j], val)
            assert np.array_equal(au[:, j], arg)
            for v in np.nonzero(~empty)[0][::7]:
                assert ae[v, j] == eid[_eid_of(g.row_ptr, g.col_idx, v, arg[v])]


@pytest.mark.parametrize("op", ["u_add_v", "u_sub_v", "u_mul_v"])
def test_sddmm_binary_complete_graph(op):
    """Elementwise u_OP_v on the complete graph = the dense broadcast X[u] OP Y[v]."""
    n, F = 23, 6
    rp = np.arange(n + 1, dtype=np.int64) * n
    ci = np.tile(np.arange(n, dtype=np.int32), n)
    X = gen.features((n, F), 53, 0).astype(np.float64)
    Y = gen.features((n, F), 53, 1).astype(np.float64)
    ref, ab = oracle.sddmm_binary(rp, ci, op, X.astype(np.float32), Y.astype(np.float32))
    fn = {"u_add_v": np.add, "u_sub_v": np.subtract, "u_mul_v": np.multiply}[op]
    dense = fn(X[None, :, :], Y[:, None, :])        # [v, u, j]
    assert np.array_equal(ref.reshape(n, n, F), dense)
    dabs = np.abs(dense) if op == "u_mul_v" else np.abs(X)[None] + np.abs(Y)[:, None]
    assert np.array_equal(ab.reshape(n, n, F), dabs)


def test_sddmm_binary_mul_sums_to_dot():
    """sum_j (u_mul_v)[e][j] = u_dot_v[e] (H = 1)."""
    g = small_graph(n=100, m=1500, seed=3)
    X = gen.features((g.n_src, 8), 55, 0)
    Y = gen.features((g.n_dst, 8), 55, 1)
    m_, _ = oracle.sddmm_binary(g.row_ptr, g.col_idx, "u_mul_v", X, Y)
    d_, _ = oracle.sddmm(g.row_ptr, g.col_idx, X, Y)
    np.testing.assert_allclose(m_.sum(axis=1), d_[:, 0], rtol=1e-12, atol=1e-13)


# ------------------------------------------------------------------ u_mul_e
def test_u_mul_e_sum_weighted_dense():
    g = small_graph()
    H, D = 3, 4
    X = gen.features((g.n_src, H * D), 21, 0)
    E = gen.features((g.nnz, H), 21, 1, gen.UNIT)
    ref, ab, _, _ = oracle.spmm(g.row_ptr, g.col_idx, "u_mul_e", "sum", X, H=H, E=E)
    for h in range(H):
        Aw = dense_adjacency(g.row_ptr, g.col_idx, g.n_src, E[:, h].astype(np.float64))
        blk = slice(h * D, (h + 1) * D)
        np.testing.assert_allclose(ref[:, blk], Aw @ X[:, blk].astype(np.float64), rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(ab[:, blk], np.abs(Aw) @ np.abs(X[:, blk].astype(np.float64)),
                                   rtol=1e-12, atol=1e-12)


def test_u_mul_e_with_eid_permutation():
    """E is indexed by edge id, not CSR position."""
    g = small_graph(n=90, m=800)
    H = 2
    X = gen.features((g.n_src, 2 * H), 4, 0)
    E = gen.features((g.nnz, H), 4, 1, gen.UNIT)
    eid = gen.permutation(g.nnz, 5).astype(np.int32)
    ref, _, _, _ = oracle.spmm(g.row_ptr, g.col_idx, "u_mul_e", "sum", X, H=H, E=E, eid=eid)
    Epos = E[eid]   # value seen at CSR position p
    ref2, _, _, _ = oracle.spmm(g.row_ptr, g.col_idx, "u_mul_e", "sum", X, H=H, E=Epos)
    assert np.array_equal(ref, ref2)


@pytest.mark.parametrize("red", ["sum", "max"])
def test_u_mul_e_ones_is_copy_u(red):
    g = small_graph()
    X = gen.features((g.n_src, 8), 23, 0)
    E = np.ones((g.nnz, 2), np.float32)
    a = oracle.spmm(g.row_ptr, g.col_idx, "u_mul_e", red, X, H=2, E=E)
    b = oracle.spmm(g.row_ptr, g.col_idx, "copy_u", red, X)
    for x, y in zip(a, b):
        if x is not None:
            assert np.array_equal(x, y)


def test_u_mul_e_max_fp32_products():
    """max compares the fp32-rounded product (numpy float32 multiply is RN)."""
    g = small_graph()
    H, D = 2, 3
    X = gen.features((g.n_src, H * D), 31, 0)
    E = gen.features((g.nnz, H), 31, 1, gen.UNIT)
    ref, _, au, ae = oracle.spmm(g.row_ptr, g.col_idx, "u_mul_e", "max", X, H=H, E=E)
    rows = edge_rows(g.row_ptr)
    M = np.full((g.n_dst, g.n_src, H * D), -np.inf)
    for h in range(H):
        prod = X[g.col_idx][:, h * D:(h + 1) * D] * E[:, h:h + 1]        # float32 RN products
        M[rows, g.col_idx, h * D:(h + 1) * D] = prod.astype(np.float64)
    A = dense_adjacency(g.row_ptr, g.col_idx, g.n_src) > 0
    val = M.max(axis=1)
    arg = M.argmax(axis=1)
    empty = ~A.any(axis=1)
    val[empty], arg[empty] = 0.0, -1
    assert np.array_equal(ref, val)
    assert np.array_equal(au, arg)


# ------------------------------------------------------------------ mlp
@pytest.mark.parametrize("regime", [gen.INT, gen.REAL])
def test_mlp_max_closed_form(regime):
    """max_u ReLU((x_u + x_v) W) == ReLU(max_u (XW)[u] + (XW)[v]) exactly in the
    reals (distributivity; ReLU(. + c) monotone).  SURVEY §8(c) pin table."""
    g = small_graph(n=150, m=2000, seed=7)
    d1, d2 = 8, 16
    if regime == gen.INT:
        X = gen.features((g.n_src, d1), 41, 0, gen.INT, lo=-8, hi=8)
        W = gen.features((d1, d2), 41, 1, gen.INT, lo=-4, hi=4)
    else:
        X = gen.features((g.n_src, d1), 41, 0)
        W = gen.features((d1, d2), 41, 1, gen.SCALED, scale=1 / np.sqrt(d1))
    ref, ab, au, ae = oracle.spmm(g.row_ptr, g.col_idx, "mlp", "max", X, W=W)
    P = X.astype(np.float64) @ W.astype(np.float64)
    A = dense_adjacency(g.row_ptr, g.col_idx, g.n_src) > 0
    Pm = np.where(A[:, :, None], P[None], -np.inf)
    best = Pm.max(axis=1)
    closed = np.maximum(best + P, 0.0)
    empty = ~A.any(axis=1)
    closed[empty] = 0.0
    if regime == gen.INT:
        assert np.array_equal(ref, closed)
        # argmax: first max of the pre-activation if positive, else the row's first edge
        first = np.array([g.col_idx[g.row_ptr[v]] if g.row_ptr[v + 1] > g.row_ptr[v] else -1
                          for v in range(g.n_dst)])
        am = Pm.argmax(axis=1)
        exp_arg = np.where(best + P > 0, am, first[:, None])
        exp_arg[empty] = -1
        assert np.array_equal(au, exp_arg)
    else:
        np.testing.assert_allclose(ref, closed, rtol=0, atol=1e-12)
    # abs-sum of the winning message: sum_k |(x_u + x_v)_k W_kj|
    v = int(np.argmax(g.degrees()))
    for j in range(d2):
        u = au[v, j]
        a = X[u].astype(np.float64) + X[v].astype(np.float64)
        assert ab[v, j] == pytest.approx(np.abs(a * W[:, j].astype(np.float64)).sum(), rel=1e-12)


def test_mlp_sum_brute_force():
    g = small_graph(n=40, m=300, seed=3)
    d1, d2 = 8, 5
    X = gen.features((g.n_src, d1), 43, 0)
    W = gen.features((d1, d2), 43, 1)
    ref, _, _, _ = oracle.spmm(g.row_ptr, g.col_idx, "mlp", "sum", X, W=W)
    for v in range(g.n_dst):
        acc = [0.0] * d2
        for p in range(g.row_ptr[v], g.row_ptr[v + 1]):
            u = g.col_idx[p]
            for i in range(d2):
                z = sum((float(X[u, k]) + float(X[v, k])) * float(W[k, i]) for k in range(d1))
                acc[i] += max(z, 0.0)
        np.testing.assert_allclose(ref[v], acc, rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("regime", [gen.INT, gen.UNIT])
def test_mlp_sum_closed_form_nonnegative(regime):
    """With X, X_dst >= 0 and W >= 0 every pre-activation is >= 0, so ReLU is the
    identity and Fig. 3b's sum aggregation is linear:
        out[v] = sum_{u in N(v)} (x_u + x_v) W = (A . (X W))[v] + deg(v) (X_dst W)[v].
    Dense A times a BLAS product -- no per-edge loop, no ReLU -- so a dropped
    x_v term, a wrong sign or a transposed W fails it.  Integer regime: exact."""
    g = small_graph(n=120, m=1500, seed=13)
    d1, d2 = 8, 24
    if regime == gen.INT:
        X = gen.features((g.n_src, d1), 44, 0, gen.INT, lo=0, hi=8)
        Xd = gen.features((g.n_dst, d1), 44, 2, gen.INT, lo=0, hi=8)
        W = gen.features((d1, d2), 44, 1, gen.INT, lo=0, hi=4)
    else:
        X = gen.features((g.n_src, d1), 44, 0, gen.UNIT)
        Xd = gen.features((g.n_dst, d1), 44, 2, gen.UNIT)
        W = gen.features((d1, d2), 44, 1, gen.UNIT)
    ref, ab, _, _ = oracle.spmm(g.row_ptr, g.col_idx, "mlp", "sum", X, W=W, X_dst=Xd)
    A = dense_adjacency(g.row_ptr, g.col_idx, g.n_src)
    XW = X.astype(np.float64) @ W.astype(np.float64)
    XdW = Xd.astype(np.float64) @ W.astype(np.float64)
    closed = A @ XW + g.degrees()[:, None] * XdW
    if regime == gen.INT:
        assert np.array_equal(ref, closed)
    else:
        np.testing.assert_allclose(ref, closed, rtol=1e-12, atol=0)
    # every term is non-negative, so the tolerance scale equals the value itself
    np.testing.assert_allclose(ab, closed, rtol=1e-12, atol=0)


def test_mlp_x_dst_separate():
    """X_dst enters only through x_v: mlp with W = I, X_dst = 0 is ReLU(copy_u max)."""
    g = small_graph(n=60, m=500, seed=8)
    d = 8
    X = gen.features((g.n_src, d), 47, 0)
    ref, _, _, _ = oracle.spmm(g.row_ptr, g.col_idx, "mlp", "max", X, W=np.eye(d, dtype=np.float32),
                               X_dst=np.zeros_like(X))
    cm, _, _, _ = oracle.spmm(g.row_ptr, g.col_idx, "copy_u", "max", X)
    assert np.array_equal(ref, np.maximum(cm, 0.0))


@pytest.mark.parametrize("key", ["mlp_max", "mlp_relu"])
def test_spec_mlp_examples(key):
    ex = GOLD[key]
    rp, ci = csr_from_edges(ex["n"], ex["edges"])
    ref, _, au, _ = oracle.spmm(rp, ci, "mlp", "max", np.array(ex["X"], np.float32),
                                W=np.array(ex["W"], np.float32))
    assert np.array_equal(ref[1], np.array(ex["expected_row1"], np.float64))
    if "expected_arg_u_row1" in ex:
        assert list(au[1]) == ex["expected_arg_u_row1"]


# ------------------------------------------------------------------ sddmm
@pytest.mark.parametrize("H,D", [(1, 7), (4, 4), (8, 2)])
def test_u_dot_v_complete_graph_is_dense(H, D):
    n = 37
    rp = np.arange(n + 1, dtype=np.int64) * n
    ci = np.tile(np.arange(n, dtype=np.int32), n)
    X = gen.features((n, H * D), 51, 0)
    Y = gen.features((n, H * D), 51, 1)
    ref, ab = oracle.sddmm(rp, ci, X, Y, H=H)
    for h in range(H):
        blk = slice(h * D, (h + 1) * D)
        dense = Y[:, blk].astype(np.float64) @ X[:, blk].astype(np.float64).T   # [v, u]
        np.testing.assert_allclose(ref[:, h].reshape(n, n), dense, rtol=1e-12, atol=1e-13)
        dabs = np.abs(Y[:, blk].astype(np.float64)) @ np.abs(X[:, blk].astype(np.float64)).T
        np.testing.assert_allclose(ab[:, h].reshape(n, n), dabs, rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("H,D", [(1, 7), (4, 4), (8, 2)])
def test_u_dot_v_e_mul_complete_graph_is_dense_hadamard(H, D):
    """u_dot_v-then-e_mul on the complete graph (self-loops included) equals the
    dense per-head (Y X^T) (.) E_dense (numpy BLAS), with a permuted edge-id map so
    E is read through eid; |terms| likewise.  Integer regime: bit-exact."""
    n = 29
    rp = np.arange(n + 1, dtype=np.int64) * n
    ci = np.tile(np.arange(n, dtype=np.int32), n)
    eid = gen.permutation(n * n, 77).astype(np.int32)
    for regime in (gen.REAL, gen.INT):
        X = gen.features((n, H * D), 52, 0, regime)
        Y = gen.features((n, H * D), 52, 1, regime)
        E = gen.features((n * n, H), 52, 2, regime, lo=-3, hi=3)
        ref, ab = oracle.sddmm_emul(rp, ci, X, Y, E, H=H, eid=eid)
        for h in range(H):
            blk = slice(h * D, (h + 1) * D)
            dense = Y[:, blk].astype(np.float64) @ X[:, blk].astype(np.float64).T        # [v, u]
            Eh = E[eid, h].astype(np.float64).reshape(n, n)                             # CSR position -> E[eid]
            dabs = np.abs(Y[:, blk].astype(np.float64)) @ np.abs(X[:, blk].astype(np.float64)).T
            if regime == gen.INT:
                assert np.array_equal(ref[:, h].reshape(n, n), dense * Eh)
            else:
                np.testing.assert_allclose(ref[:, h].reshape(n, n), dense * Eh, rtol=1e-12, atol=1e-13)
            np.testing.assert_allclose(ab[:, h].reshape(n, n), dabs * np.abs(Eh), rtol=1e-12, atol=1e-13)


def test_u_dot_v_e_mul_special_cases():
    """E == 1 gives the plain score (Eq. (4)); E == 0 gives +-0; a single edge
    with hand-computed values (2*3 + 1*(-4)) * 0.5 = 1."""
    g = small_graph()
    X = gen.features((g.n_src, 8), 53, 0)
    ones = np.ones((g.nnz, 2), np.float32)
    r1, a1 = oracle.sddmm_emul(g.row_ptr, g.col_idx, X, X, ones, H=2)
    r0, a0 = oracle.sddmm(g.row_ptr, g.col_idx, X, X, H=2)
    assert np.array_equal(r1, r0) and np.array_equal(a1, a0)
    rz, az = oracle.sddmm_emul(g.row_ptr, g.col_idx, X, X, np.zeros((g.nnz, 2), np.float32), H=2)
    assert (rz == 0).all() and (az == 0).all()
    rp, ci = csr_from_edges(2, [[0, 1]])
    X2 = np.array([[2, 1], [3, -4]], np.float32)
    r, _ = oracle.sddmm_emul(rp, ci, X2, X2, np.array([[0.5]], np.float32), H=1)
    assert r.tolist() == [[1.0]]


def test_spec_dot_examples():
    ex = GOLD["dot"]
    rp, ci = csr_from_edges(ex["n"], ex["edges"])
    ref, _ = oracle.sddmm(rp, ci, np.array(ex["X"], np.float32))
    assert ref.tolist() == ex["expected"]
    ex = GOLD["orthogonal_dot"]
    rp, ci = csr_from_edges(ex["n"], ex["edges"])
    ref, _ = oracle.sddmm(rp, ci, np.array(ex["X"], np.float32))
    assert ref.tolist() == ex["expected"]
    ex = GOLD["multi_head_dot"]
    rp, ci = csr_from_edges(2, [[0, 1]])
    X = np.zeros((2, 6), np.float32)
    X[0] = np.array(ex["src"], np.float32).reshape(-1)
    X[1] = np.array(ex["dst"], np.float32).reshape(-1)
    ref, _ = oracle.sddmm(rp, ci, X, H=ex["H"])
    assert ref[0].tolist() == ex["expected"]


def test_sddmm_rows_subset_matches_full():
    g = small_graph()
    X = gen.features((g.n_src, 8), 53, 0)
    full, _ = oracle.sddmm(g.row_ptr, g.col_idx, X, H=2)
    rows = np.array([5, 0, 100, 3], np.int64)
    sub, _ = oracle.sddmm(g.row_ptr, g.col_idx, X, H=2, rows=rows)
    assert np.array_equal(sub, full[oracle.edge_positions(g.row_ptr, rows)])


@pytest.mark.parametrize("regime", [gen.INT, gen.REAL])
def test_adjoint_identity(regime):
    """Gradient duality: <G, spmm_{u_mul_e,sum}(A, X, a)> ==
    <a, sddmm_{u_dot_v}(X_src = X, Y_dst = G)>, per head."""
    g = small_graph()
    H, D = 2, 4
    lo, hi = -5, 5
    X = gen.features((g.n_src, H * D), 61, 0, regime, lo=lo, hi=hi)
    G = gen.features((g.n_dst, H * D), 61, 1, regime, lo=lo, hi=hi)
    a = gen.features((g.nnz, H), 61, 2, gen.INT if regime == gen.INT else gen.UNIT, lo=0, hi=4)
    out, _, _, _ = oracle.spmm(g.row_ptr, g.col_idx, "u_mul_e", "sum", X, H=H, E=a)
    s, _ = oracle.sddmm(g.row_ptr, g.col_idx, X, G, H=H)
    lhs = float((G.astype(np.float64) * out).sum())
    rhs = float((a.astype(np.float64) * s).sum())
    if regime == gen.INT:
        assert lhs == rhs
    else:
        assert lhs == pytest.approx(rhs, rel=1e-12, abs=1e-9)


# ------------------------------------------------------------------ edge softmax
def test_edge_softmax_invariants():
    g = small_graph()
    H = 4
    S = gen.features((g.nnz, H), 71, 0)
    al = oracle.edge_softmax(g.row_ptr, S, H=H)
    rows = edge_rows(g.row_ptr)
    sums = np.zeros((g.n_dst, H))
    np.add.at(sums, rows, al)
    nonempty = g.degrees() > 0
    np.testing.assert_allclose(sums[nonempty], 1.0, rtol=0, atol=1e-13)
    # shift invariance s -> s + c_v
    c = gen.features((g.n_dst,), 71, 1, gen.INT, lo=-3, hi=3)
    al2 = oracle.edge_softmax(g.row_ptr, S + c[rows][:, None], H=H)
    np.testing.assert_allclose(al2, al, rtol=1e-6, atol=0)
    # constant scores -> 1/deg; degree-1 rows -> exactly 1
    al3 = oracle.edge_softmax(g.row_ptr, np.full((g.nnz, H), 0.25, np.float32), H=H)
    np.testing.assert_allclose(al3, 1.0 / g.degrees()[rows][:, None] * np.ones((1, H)), rtol=1e-15)
    d1 = g.degrees()[rows] == 1
    assert (al[d1] == 1.0).all()


def test_edge_softmax_matches_torch_dense():
    import torch
    g = small_graph(n=64, m=700, seed=12)
    H = 2
    S = gen.features((g.nnz, H), 73, 0) * 4
    eid = gen.permutation(g.nnz, 3).astype(np.int32)
    al = oracle.edge_softmax(g.row_ptr, S, H=H, eid=eid)
    rows = edge_rows(g.row_ptr)
    for h in range(H):
        M = torch.full((g.n_dst, g.n_src), float("-inf"), dtype=torch.float64)
        M[torch.from_numpy(rows), torch.from_numpy(g.col_idx.astype(np.int64))] = \
            torch.from_numpy(S[eid, h].astype(np.float64))
        P = torch.softmax(M, dim=1)
        got = P[torch.from_numpy(rows), torch.from_numpy(g.col_idx.astype(np.int64))].numpy()
        np.testing.assert_allclose(al[:, h], got, rtol=1e-12, atol=0)


# ------------------------------------------------------------------ fused GAT definition
def test_gat_oracle_vs_torch_dense_attention():
    """or_gat == dense masked softmax attention per head (torch, fp64)."""
    import torch
    g = small_graph(n=80, m=900, seed=14)
    H, D = 2, 4
    X = gen.features((g.n_src, H * D), 81, 0)
    Y = gen.features((g.n_dst, H * D), 81, 1)
    ref, ab = oracle.gat(g.row_ptr, g.col_idx, X, Y, H=H)
    A = torch.from_numpy(dense_adjacency(g.row_ptr, g.col_idx, g.n_src) > 0)
    for h in range(H):
        xs = torch.from_numpy(X[:, h * D:(h + 1) * D].astype(np.float64))
        ys = torch.from_numpy(Y[:, h * D:(h + 1) * D].astype(np.float64))
        S = (ys @ xs.T).masked_fill(~A, float("-inf"))
        P = torch.softmax(S, dim=1).nan_to_num(0.0)      # empty rows -> 0
        np.testing.assert_allclose(ref[:, h * D:(h + 1) * D], (P @ xs).numpy(), rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(ab[:, h * D:(h + 1) * D], (P @ xs.abs()).numpy(), rtol=1e-12, atol=1e-13)


def test_gat_oracle_zero_query_is_mean():
    """Y = 0 -> every score 0 -> alpha = 1/deg -> out = mean of in-neighbour features."""
    g = small_graph(n=70, m=600, seed=15)
    X = gen.features((g.n_src, 8), 82, 0)
    ref, _ = oracle.gat(g.row_ptr, g.col_idx, X, np.zeros((g.n_dst, 8), np.float32), H=2)
    A = dense_adjacency(g.row_ptr, g.col_idx, g.n_src)
    deg = np.maximum(A.sum(1, keepdims=True), 1)
    np.testing.assert_allclose(ref, (A @ X.astype(np.float64)) / deg, rtol=1e-12, atol=1e-14)
