"""Pins for the oracle's backward routines (gradient duality):
each is compared with torch autograd (float64) of a dense formulation of the
forward op on small graphs -- an independent computation of the same gradient."""
import numpy as np
import pytest
import torch

import gen
import oracle
from helpers import dense_adjacency, edge_rows


def graph(n=60, m=500, seed=2):
    return gen.random_graph(n, m, seed, sigma=1.2, n_empty=3)


def t64(a):
    return torch.from_numpy(np.asarray(a, np.float64))


@pytest.mark.parametrize("op", ["copy_u", "u_mul_e"])
def test_spmm_sum_backward_vs_autograd(op):
    g = graph()
    H, D = 2, 3
    X = gen.features((g.n_src, H * D), 1, 0)
    E = gen.features((g.nnz, H), 1, 1, gen.UNIT)
    G = gen.features((g.n_dst, H * D), 1, 2)
    dX, dE = oracle.spmm_backward(g.row_ptr, g.col_idx, op, "sum", X, G, n_src=g.n_src, H=H,
                                  E=E if op == "u_mul_e" else None, want_dE=op == "u_mul_e")
    Xt = t64(X).requires_grad_()
    Et = t64(E).requires_grad_()
    out = torch.zeros(g.n_dst, H * D, dtype=torch.float64)
    rows = torch.from_numpy(edge_rows(g.row_ptr))
    cols = torch.from_numpy(g.col_idx.astype(np.int64))
    msg = Xt[cols]
    if op == "u_mul_e":
        msg = msg * Et.repeat_interleave(D, dim=1)
    out = out.index_add(0, rows, msg)
    (out * t64(G)).sum().backward()
    np.testing.assert_allclose(dX, Xt.grad.numpy(), rtol=1e-12, atol=1e-12)
    if op == "u_mul_e":
        np.testing.assert_allclose(dE, Et.grad.numpy(), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("op", ["copy_u", "u_mul_e"])
def test_spmm_max_backward_vs_autograd(op):
    g = graph(seed=4)
    H, D = 2, 2
    X = gen.features((g.n_src, H * D), 3, 0)          # real regime: no ties
    E = gen.features((g.nnz, H), 3, 1, gen.UNIT)
    G = gen.features((g.n_dst, H * D), 3, 2)
    _, _, au, _ = oracle.spmm(g.row_ptr, g.col_idx, op, "max", X, H=H, E=E if op == "u_mul_e" else None)
    dX, dE = oracle.spmm_backward(g.row_ptr, g.col_idx, op, "max", X, G, n_src=g.n_src, H=H,
                                  E=E if op == "u_mul_e" else None, arg_u=au, want_dE=op == "u_mul_e")
    Xt = t64(X).requires_grad_()
    Et = t64(E).requires_grad_()
    rows = edge_rows(g.row_ptr)
    M = torch.full((g.n_dst, g.n_src, H * D), float("-inf"), dtype=torch.float64)
    msg = Xt[torch.from_numpy(g.col_idx.astype(np.int64))]
    if op == "u_mul_e":
        msg = msg * Et.repeat_interleave(D, dim=1)
    M = M.index_put((torch.from_numpy(rows), torch.from_numpy(g.col_idx.astype(np.int64))), msg)
    out = M.max(dim=1).values
    nonempty = torch.from_numpy(np.diff(g.row_ptr) > 0)
    (out[nonempty] * t64(G)[nonempty]).sum().backward()
    np.testing.assert_allclose(dX, Xt.grad.numpy(), rtol=1e-12, atol=1e-12)
    if op == "u_mul_e":
        np.testing.assert_allclose(dE, Et.grad.numpy(), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("op", ["copy_u", "u_mul_e"])
def test_spmm_min_backward_vs_autograd(op):
    g = graph(seed=8)
    H, D = 2, 2
    X = gen.features((g.n_src, H * D), 5, 0)
    E = gen.features((g.nnz, H), 5, 1, gen.UNIT)
    G = gen.features((g.n_dst, H * D), 5, 2)
    Eo = E if op == "u_mul_e" else None
    _, _, au, _ = oracle.spmm(g.row_ptr, g.col_idx, op, "min", X, H=H, E=Eo)
    dX, dE = oracle.spmm_backward(g.row_ptr, g.col_idx, op, "min", X, G, n_src=g.n_src, H=H, E=Eo, arg_u=au,
                                  want_dE=op == "u_mul_e")
    Xt = t64(X).requires_grad_()
    Et = t64(E).requires_grad_()
    rows = edge_rows(g.row_ptr)
    M = torch.full((g.n_dst, g.n_src, H * D), float("inf"), dtype=torch.float64)
    msg = Xt[torch.from_numpy(g.col_idx.astype(np.int64))]
    if op == "u_mul_e":
        msg = msg * Et.repeat_interleave(D, dim=1)
    M = M.index_put((torch.from_numpy(rows), torch.from_numpy(g.col_idx.astype(np.int64))), msg)
    out = M.min(dim=1).values
    nonempty = torch.from_numpy(np.diff(g.row_ptr) > 0)
    (out[nonempty] * t64(G)[nonempty]).sum().backward()
    np.testing.assert_allclose(dX, Xt.grad.numpy(), rtol=1e-12, atol=1e-12)
    if op == "u_mul_e":
        np.testing.assert_allclose(dE, Et.grad.numpy(), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("op", ["copy_u", "u_mul_e"])
def test_spmm_mean_backward_vs_autograd(op):
    g = graph(seed=10)
    H, D = 2, 3
    X = gen.features((g.n_src, H * D), 7, 0)
    E = gen.features((g.nnz, H), 7, 1, gen.UNIT)
    G = gen.features((g.n_dst, H * D), 7, 2)
    Eo = E if op == "u_mul_e" else None
    dX, dE = oracle.spmm_backward(g.row_ptr, g.col_idx, op, "mean", X, G, n_src=g.n_src, H=H, E=Eo,
                                  want_dE=op == "u_mul_e")
    Xt = t64(X).requires_grad_()
    Et = t64(E).requires_grad_()
    rows = torch.from_numpy(edge_rows(g.row_ptr))
    msg = Xt[torch.from_numpy(g.col_idx.astype(np.int64))]
    if op == "u_mul_e":
        msg = msg * Et.repeat_interleave(D, dim=1)
    out = torch.zeros(g.n_dst, H * D, dtype=torch.float64).index_add(0, rows, msg)
    deg = torch.from_numpy(np.maximum(np.diff(g.row_ptr), 1).astype(np.float64))[:, None]
    ((out / deg) * t64(G)).sum().backward()
    np.testing.assert_allclose(dX, Xt.grad.numpy(), rtol=1e-12, atol=1e-12)
    if op == "u_mul_e":
        np.testing.assert_allclose(dE, Et.grad.numpy(), rtol=1e-12, atol=1e-12)


def test_sddmm_backward_vs_autograd():
    g = graph(seed=6)
    H, D = 2, 4
    X = gen.features((g.n_src, H * D), 5, 0)
    Y = gen.features((g.n_dst, H * D), 5, 1)
    dS = gen.features((g.nnz, H), 5, 2)
    dX, dY = oracle.sddmm_backward(g.row_ptr, g.col_idx, X, Y, dS, H=H)
    Xt, Yt = t64(X).requires_grad_(), t64(Y).requires_grad_()
    rows = torch.from_numpy(edge_rows(g.row_ptr))
    cols = torch.from_numpy(g.col_idx.astype(np.int64))
    s = (Xt[cols].view(-1, H, D) * Yt[rows].view(-1, H, D)).sum(-1)
    (s * t64(dS)).sum().backward()
    np.testing.assert_allclose(dX, Xt.grad.numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(dY, Yt.grad.numpy(), rtol=1e-12, atol=1e-12)


def test_edge_softmax_backward_vs_autograd():
    g = graph(seed=8)
    H = 3
    S = gen.features((g.nnz, H), 7, 0) * 3
    dA = gen.features((g.nnz, H), 7, 1)
    alpha = oracle.edge_softmax(g.row_ptr, S, H=H).astype(np.float32)
    ds = oracle.edge_softmax_backward(g.row_ptr, alpha, dA, H=H)
    St = t64(S).requires_grad_()
    rows = torch.from_numpy(edge_rows(g.row_ptr))
    cols = torch.from_numpy(g.col_idx.astype(np.int64))
    M = torch.full((g.n_dst, g.n_src, H), float("-inf"), dtype=torch.float64)
    M = M.index_put((rows, cols), St)
    A = torch.softmax(M, dim=1)[rows, cols]
    (A * t64(dA)).sum().backward()
    # oracle uses the fp32-rounded alpha; tolerance covers that rounding
    np.testing.assert_allclose(ds, St.grad.numpy(), rtol=1e-6, atol=1e-7)
