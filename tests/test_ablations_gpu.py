"""Parity of the ablation paths the measurements compare against the product
kernels (SURVEY §8(f) f3 / the paper's E6 and E7 ablations), forced per
handle with fg_graph_tune, against the oracle:

  * hybrid partitioning (E7 P:875-877): the hottest
    sources staged in shared memory for copy_u-sum -- bit-identical to the
    plain kernel (same values, same order), on both the group-per-row and the
    CTA-per-row paths, and untouched when the table was built for another width;
  * thread-per-edge dot products for gSDDMM (E6) -- within
    1e-4 * sum|terms| (its per-edge summation order differs);
  * the MLP ablations (FFMA, bf16 2-split) on the regular MLP tests' inputs.
"""
import numpy as np
import pytest
import torch

import gen
import oracle
from helpers import check_close, tuned

pytestmark = pytest.mark.gpu
TOL = 1e-4


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.fixture(scope="module")
def skew(cuda_ok):
    import paper_2008_11359_b200 as fgp
    g = gen.random_graph(4000, 160000, 61, sigma=1.6, n_empty=40)
    return g, fgp.Graph(dev(g.row_ptr), dev(g.col_idx))


@pytest.mark.parametrize("F", [16, 32, 128])
@pytest.mark.parametrize("smem_kb", [8, 48, 96])
def test_hybrid_copy_u_sum_bit_identical(skew, F, smem_kb):
    import paper_2008_11359_b200 as fgp
    g, G = skew
    X = gen.features((g.n_src, F), 1400 + F, 0, gen.REAL)
    Xd = dev(X)
    plain = fgp.spmm(G, "copy_u", "sum", Xd)
    G.prepare_hybrid(F * 4, smem_kb * 1024)
    k, share = G.hybrid_info()
    assert k == min(g.n_src, smem_kb * 1024 // (F * 4)) and 0 < share <= 1
    deg_out = np.bincount(g.col_idx, minlength=g.n_src)
    assert share == pytest.approx(np.sort(deg_out)[::-1][:k].sum() / g.nnz)   # the k hottest sources
    with tuned(G, hybrid=1):
        hyb = fgp.spmm(G, "copy_u", "sum", Xd)
        with tuned(G, spmm_heavy_deg=64):           # CTA-per-row rows inside the persistent loop
            hyb_h = fgp.spmm(G, "copy_u", "sum", Xd)
        with tuned(G, spmm_heavy_deg=64, hybrid=0):
            plain_h = fgp.spmm(G, "copy_u", "sum", Xd)
        # a width the table was not built for runs the plain kernel
        X2 = dev(gen.features((g.n_src, 2 * F), 1401, 0, gen.REAL))
        other = fgp.spmm(G, "copy_u", "sum", X2)
    assert torch.equal(hyb, plain)
    assert torch.equal(hyb_h, plain_h)
    ref, ab, _, _ = oracle.spmm(g.row_ptr, g.col_idx, "copy_u", "sum", X)
    check_close(hyb.cpu().numpy(), ref, ab, TOL, f"hybrid copy_u-sum F={F}")
    assert torch.equal(other, fgp.spmm(G, "copy_u", "sum", X2))


@pytest.mark.parametrize("H,D", [(1, 16), (1, 128), (1, 512), (8, 32), (4, 4)])
@pytest.mark.parametrize("use_eid", [False, True])
def test_sddmm_thread_per_edge(skew, H, D, use_eid):
    import paper_2008_11359_b200 as fgp
    g, G0 = skew
    eid = gen.permutation(g.nnz, 17).astype(np.int32) if use_eid else None
    G = fgp.Graph(dev(g.row_ptr), dev(g.col_idx), eid=None if eid is None else dev(eid)) if use_eid else G0
    X = gen.features((g.n_src, H * D), 1450 + D, 0, gen.REAL)
    Y = gen.features((g.n_dst, H * D), 1451 + D, 0, gen.REAL)
    with tuned(G, sddmm_dot=1):
        out = fgp.sddmm(G, dev(X), dev(Y), H=H).cpu().numpy()
        E = gen.features((g.nnz, H), 1452, 0, gen.UNIT)
        oe = fgp.sddmm(G, dev(X), dev(Y), H=H, E=dev(E)).cpu().numpy()
    ref, ab = oracle.sddmm(g.row_ptr, g.col_idx, X, Y, H=H)
    pos = np.arange(g.nnz) if eid is None else eid
    check_close(out[pos], ref, ab, TOL, f"thread-per-edge u_dot_v H={H} D={D}")
    re_, rab = oracle.sddmm_emul(g.row_ptr, g.col_idx, X, Y, E, H=H, eid=eid)
    check_close(oe[pos], re_, rab, TOL, f"thread-per-edge u_dot_v e_mul H={H} D={D}")
