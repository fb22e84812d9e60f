"""Multi-GPU path on one GPU:
  * shard simulator: each rank's local graph (dst-row range, global source ids)
    runs the unchanged kernels; concatenated outputs are bit-identical to the
    unsharded run (per-row computation depends only on the row);
  * fg_allgather_rows through a real 1-rank NCCL communicator."""
import numpy as np
import pytest
import torch

import gen
from paper_2008_11359_b200.shard import make_shard

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.fixture(scope="module")
def graph(cuda_ok):
    return gen.random_graph(4000, 200000, 31, sigma=1.5, n_empty=40)


@pytest.mark.parametrize("P", [2, 3, 8])
def test_shard_simulator_bit_identical(graph, P):
    import paper_2008_11359_b200 as fgp
    g = graph
    F, H = 256, 8
    X = dev(gen.features((g.n_src, F), 7, 0))
    X8 = dev(gen.features((g.n_src, 8), 7, 1))
    W = dev(gen.features((8, 128), 7, 2, gen.SCALED, scale=0.35))
    G = fgp.Graph(dev(g.row_ptr), dev(g.col_idx))
    full_sum = fgp.spmm(G, "copy_u", "sum", X)
    full_max, full_au, _ = fgp.spmm(G, "copy_u", "max", X, arg_u=True)
    full_s = fgp.sddmm(G, X, H=H)
    full_a = fgp.edge_softmax(G, full_s, H=H)
    full_o = fgp.spmm(G, "u_mul_e", "sum", X, H=H, E=full_a)
    full_m, full_mau, _ = fgp.spmm(G, "mlp", "max", X8, W=W, arg_u=True)
    parts = {k: [] for k in ("sum", "max", "au", "s", "o", "m", "mau")}
    for r in range(P):
        sh = make_shard(g.row_ptr, g.col_idx, r, P)
        L = fgp.Graph(dev(sh.row_ptr), dev(sh.col_idx), n_src=g.n_src)
        Y = X[sh.lo:sh.hi]
        parts["sum"].append(fgp.spmm(L, "copy_u", "sum", X))
        m, au, _ = fgp.spmm(L, "copy_u", "max", X, arg_u=True)
        parts["max"].append(m)
        parts["au"].append(au)
        s = fgp.sddmm(L, X, Y, H=H)
        parts["s"].append(s)
        a = fgp.edge_softmax(L, s, H=H)
        parts["o"].append(fgp.spmm(L, "u_mul_e", "sum", X, H=H, E=a))
        mm, mau, _ = fgp.spmm(L, "mlp", "max", X8, W=W, X_dst=X8[sh.lo:sh.hi], arg_u=True)
        parts["m"].append(mm)
        parts["mau"].append(mau)
    cat = {k: torch.cat(v) for k, v in parts.items()}
    assert torch.equal(cat["sum"], full_sum)
    assert torch.equal(cat["max"], full_max) and torch.equal(cat["au"], full_au)
    assert torch.equal(cat["s"], full_s)
    assert torch.equal(cat["o"], full_o)
    assert torch.equal(cat["m"], full_m) and torch.equal(cat["mau"], full_mau)


def test_allgather_rows_single_rank_nccl(cuda_ok):
    import paper_2008_11359_b200 as fgp
    uid = fgp.comm_unique_id()
    c = fgp.Comm(uid, 1, 0)
    n, F = 1000, 64
    X = torch.randn(n, F, device="cuda")
    full = torch.zeros_like(X)
    c.allgather_rows([0, n], X, full)
    torch.cuda.synchronize()
    assert torch.equal(full, X)
    # in place (local block inside the full buffer)
    full2 = X.clone()
    c.allgather_rows([0, n], full2, full2)
    torch.cuda.synchronize()
    assert torch.equal(full2, X)
    c.close()


def test_bench_step_overlapped_allgather_single_rank(cuda_ok):
    """bench.Step's N > 1 schedule (all-gathers on their own stream, each op
    waiting only for the tensor it reads) through a real 1-rank NCCL
    communicator on a shard that is the whole graph: two steps back to back give
    the same outputs as the unsharded step (the second step's gathers must wait
    for the first step's ops)."""
    import bench
    import paper_2008_11359_b200 as fgp
    from paper_2008_11359_b200.shard import make_shard
    g = gen.random_graph(3000, 150000, 41, sigma=1.4, n_empty=20)
    host = bench.make_inputs(g)
    ref_stream = torch.cuda.Stream()
    R = bench.Step(g, None, host, None, ref_stream)
    with torch.cuda.stream(ref_stream):
        R.enqueue()
    torch.cuda.synchronize()
    c = fgp.Comm(fgp.comm_unique_id(), 1, 0)
    st = torch.cuda.Stream()
    S = bench.Step(g, make_shard(g.row_ptr, g.col_idx, 0, 1), host, c, st)
    with torch.cuda.stream(st):
        S.enqueue()
        S.enqueue()
    torch.cuda.synchronize()
    for a, b in zip(S.outputs(), R.outputs()):
        assert torch.equal(a, b)
    c.close()


def test_bench_e2e_pipeline_matches_step(cuda_ok):
    """bench.py's end-to-end schedule (inputs from pinned host buffers on a copy
    stream, reordered ops, the GAT aggregation on two row-half graph handles,
    results shipped to pinned host buffers on a second copy stream) returns
    exactly the outputs of the plain device step."""
    import bench
    g = gen.random_graph(3000, 150000, 43, sigma=1.4, n_empty=20)
    host = bench.make_inputs(g)
    st = torch.cuda.Stream()
    S = bench.Step(g, None, host, None, st)
    with torch.cuda.stream(st):
        S.enqueue()
    torch.cuda.synchronize()
    ref = [o.clone() for o in S.outputs()]
    for o in S.outputs():
        o.fill_(-7.0) if o.is_floating_point() else o.fill_(-7)
    ins = {k: torch.from_numpy(np.ascontiguousarray(host[k])).pin_memory() for k in ("X512", "X256", "X128", "X8")}
    w_h = torch.from_numpy(host["W"]).pin_memory()
    outs_h = {id(o): torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in S.outputs()}
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(st):
        h2d.wait_stream(st)
        d2h.wait_stream(st)
        S.enqueue_pipelined(ins, w_h, outs_h, h2d, d2h)
        st.wait_stream(d2h)
    torch.cuda.synchronize()
    for o, r in zip(S.outputs(), ref):
        assert torch.equal(outs_h[id(o)], r.cpu())


def test_dist_spmm_sddmm_single_rank(cuda_ok, graph):
    """fg_dist_spmm / fg_dist_sddmm through a 1-rank NCCL communicator (the shard
    is the whole graph): the all-gather fills X_full from a separate X_local and
    the local ops equal the unsharded fg_spmm / fg_sddmm bit for bit."""
    import paper_2008_11359_b200 as fgp
    g = graph
    G = fgp.Graph(dev(g.row_ptr), dev(g.col_idx))
    c = fgp.Comm(fgp.comm_unique_id(), 1, 0)
    off = [0, g.n_dst]
    H, D = 8, 32
    X = dev(gen.features((g.n_src, H * D), 17, 0))
    E = dev(gen.features((g.nnz, H), 17, 1, gen.UNIT))
    Xf = torch.zeros_like(X)
    o = c.dist_spmm(G, off, "copy_u", "sum", X, Xf)
    torch.cuda.synchronize()
    assert torch.equal(Xf, X)
    assert torch.equal(o, fgp.spmm(G, "copy_u", "sum", X))
    Xf.zero_()
    o = c.dist_spmm(G, off, "u_mul_e", "sum", X, Xf, H=H, E=E)
    assert torch.equal(o, fgp.spmm(G, "u_mul_e", "sum", X, H=H, E=E))
    Xf.zero_()
    s = c.dist_sddmm(G, off, X, Xf, X, H=H)
    assert torch.equal(s, fgp.sddmm(G, X, H=H))
    c.close()
