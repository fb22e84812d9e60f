"""Destination-row sharding on CPU: offsets, local CSR with
global source ids, and a world_size-2 gloo run of the sharded step (all-gather
of X row blocks + local aggregation) whose concatenated outputs must equal the
unsharded result bit for bit.  The GPU side of the same logic is
tests/test_dist_gpu.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle
from paper_2008_11359_b200.shard import make_shard, nnz_balanced_offsets


def test_offsets_balanced_and_cover():
    g = gen.random_graph(1000, 40000, 3, sigma=1.5, n_empty=20)
    for P in (1, 2, 3, 4, 8):
        off = nnz_balanced_offsets(g.row_ptr, P)
        assert off[0] == 0 and off[-1] == g.n_dst and (np.diff(off) >= 0).all()
        nnz = np.diff(g.row_ptr[off])
        assert nnz.sum() == g.nnz
        assert nnz.max() <= g.nnz / P + g.degrees().max()   # within one row of the ideal split


def test_local_csr_keeps_global_ids():
    g = gen.random_graph(300, 5000, 4, n_empty=5)
    P = 3
    parts = [make_shard(g.row_ptr, g.col_idx, r, P) for r in range(P)]
    assert np.array_equal(np.concatenate([p.col_idx for p in parts]), g.col_idx)
    for p in parts:
        assert p.row_ptr[0] == 0 and p.nnz == g.row_ptr[p.hi] - g.row_ptr[p.lo]
        assert np.array_equal(p.row_ptr + p.edge_lo, g.row_ptr[p.lo:p.hi + 1])


def test_degenerate_more_ranks_than_rows():
    rp = np.array([0, 2, 3], np.int64)
    off = nnz_balanced_offsets(rp, 4)
    assert off[0] == 0 and off[-1] == 2 and (np.diff(off) >= 0).all()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = gen.random_graph(400, 9000, 21, sigma=1.4, n_empty=10)
    F = 12
    X = gen.features((g.n_src, F), 5, 0, gen.INT)
    sh = make_shard(g.row_ptr, g.col_idx, rank, world)
    # all-gather-v of row blocks, as fg_allgather_rows does over NCCL: one
    # broadcast per root of that root's block; only this rank's block is local
    blocks = [torch.zeros((int(sh.offsets[r + 1] - sh.offsets[r]), F)) for r in range(world)]
    blocks[rank].copy_(torch.from_numpy(np.ascontiguousarray(X[sh.lo:sh.hi])))
    for r in range(world):
        dist.broadcast(blocks[r], src=r)
    X_full = torch.cat(blocks).numpy()
    out, _, _, _ = oracle.spmm(sh.row_ptr, sh.col_idx, "copy_u", "sum", X_full)
    mx, _, au, _ = oracle.spmm(sh.row_ptr, sh.col_idx, "copy_u", "max", X_full)
    s, _ = oracle.sddmm(sh.row_ptr, sh.col_idx, X_full, X_full[sh.lo:sh.hi])
    res = [None] * world
    dist.all_gather_object(res, (out, mx, au, s))
    if rank == 0:
        ref, _, _, _ = oracle.spmm(g.row_ptr, g.col_idx, "copy_u", "sum", X)
        rmx, _, rau, _ = oracle.spmm(g.row_ptr, g.col_idx, "copy_u", "max", X)
        rs, _ = oracle.sddmm(g.row_ptr, g.col_idx, X)
        ok = (np.array_equal(np.concatenate([r[0] for r in res]), ref)
              and np.array_equal(np.concatenate([r[1] for r in res]), rmx)
              and np.array_equal(np.concatenate([r[2] for r in res]), rau)
              and np.array_equal(np.concatenate([r[3] for r in res]), rs))
        q.put(ok)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_step_matches_unsharded(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) is True
