"""GPU backward kernels (gradient duality) vs the fp64 oracle
backward (itself pinned to torch autograd in tests/test_oracle_backward.py)."""
import numpy as np
import pytest
import torch

import gen
import oracle
from helpers import check_close

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.fixture(scope="module")
def G(cuda_ok):
    import paper_2008_11359_b200 as fgp
    g = gen.random_graph(2000, 60000, 91, sigma=1.5, n_empty=30)
    h = fgp.Graph(dev(g.row_ptr), dev(g.col_idx))
    return g, h, h.transpose()


def test_transpose_is_csc(G):
    g, h, hT = G
    assert (hT.n_dst, hT.n_src, hT.nnz) == (g.n_src, g.n_dst, g.nnz)
    import paper_2008_11359_b200 as fgp
    # copy_u sum over gT of ones == out-degree
    ones = torch.ones((g.n_dst, 4), device="cuda")
    outdeg = fgp.spmm(hT, "copy_u", "sum", ones).cpu().numpy()[:, 0]
    assert np.array_equal(outdeg, np.bincount(g.col_idx, minlength=g.n_src).astype(np.float32))


@pytest.mark.parametrize("op", ["copy_u", "u_mul_e"])
@pytest.mark.parametrize("red", ["sum", "max", "min", "mean"])
def test_spmm_backward(G, op, red):
    import paper_2008_11359_b200 as fgp
    g, h, hT = G
    H, D = 4, 8
    F = H * D
    X = gen.features((g.n_src, F), 21, 0)
    E = gen.features((g.nnz, H), 21, 1, gen.UNIT)
    dOut = gen.features((g.n_dst, F), 21, 2)
    Ed = dev(E) if op == "u_mul_e" else None
    arg_u = rau = None
    if red in ("max", "min"):
        _, au, _ = fgp.spmm(h, op, red, dev(X), H=H, E=Ed, arg_u=True, arg_e=True)
        arg_u = au
        # the oracle side uses the oracle's own winners; they must match the kernel's
        _, _, rau, _ = oracle.spmm(g.row_ptr, g.col_idx, op, red, X, H=H, E=E if op == "u_mul_e" else None)
        assert np.array_equal(au.cpu().numpy(), rau)
    dX, dE = fgp.spmm_backward(h, hT, op, red, dev(dOut), H=H, X=dev(X), E=Ed, arg_u=arg_u,
                               want_dE=op == "u_mul_e")
    rdX, rdE = oracle.spmm_backward(g.row_ptr, g.col_idx, op, red, X, dOut, n_src=g.n_src, H=H,
                                    E=E if op == "u_mul_e" else None, arg_u=rau, want_dE=op == "u_mul_e")
    # tolerance scale: the same gradient of |inputs|
    bdX, bdE = oracle.spmm_backward(g.row_ptr, g.col_idx, op, red, np.abs(X), np.abs(dOut), n_src=g.n_src, H=H,
                                    E=np.abs(E) if op == "u_mul_e" else None, arg_u=rau,
                                    want_dE=op == "u_mul_e")
    check_close(dX.cpu().numpy(), rdX, bdX, 1e-4, f"dX {op}-{red}")
    if op == "u_mul_e":
        check_close(dE.cpu().numpy(), rdE, bdE, 1e-4, f"dE {op}-{red}")


def test_sddmm_backward(G):
    import paper_2008_11359_b200 as fgp
    g, h, hT = G
    H, D = 8, 4
    X = gen.features((g.n_src, H * D), 31, 0)
    Y = gen.features((g.n_dst, H * D), 31, 1)
    dS = gen.features((g.nnz, H), 31, 2)
    dX, dY = fgp.sddmm_backward(h, hT, dev(X), dev(Y), dev(dS), H=H)
    rdX, rdY = oracle.sddmm_backward(g.row_ptr, g.col_idx, X, Y, dS, H=H)
    bdX, bdY = oracle.sddmm_backward(g.row_ptr, g.col_idx, np.abs(X), np.abs(Y), np.abs(dS), H=H)
    check_close(dX.cpu().numpy(), rdX, bdX, 1e-4, "sddmm dX")
    check_close(dY.cpu().numpy(), rdY, bdY, 1e-4, "sddmm dY")


@pytest.mark.parametrize("H", [1, 8, 3, 4, 16, 128])
def test_edge_softmax_backward(G, H):
    import paper_2008_11359_b200 as fgp
    g, h, hT = G
    S = gen.features((g.nnz, H), 41, 0) * 4
    dA = gen.features((g.nnz, H), 41, 1)
    # alpha from the oracle's forward (rounded to fp32) feeds both sides
    alpha32 = oracle.edge_softmax(g.row_ptr, S, H=H).astype(np.float32)
    ds = fgp.edge_softmax_backward(h, dev(alpha32), dev(dA), H=H).cpu().numpy()
    ref = oracle.edge_softmax_backward(g.row_ptr, alpha32, dA, H=H)
    # |terms|: alpha*|dalpha| + alpha * sum alpha*|dalpha|
    a = alpha32.astype(np.float64)
    bound = oracle.edge_softmax_backward(g.row_ptr, a.astype(np.float32), np.abs(dA), H=H)
    bound = np.abs(bound) + 2 * a * np.abs(dA)
    check_close(ds, ref, bound, 1e-4, f"softmax backward H={H}")
