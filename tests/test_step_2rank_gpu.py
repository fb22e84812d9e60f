"""The sharded bench step (bench.Step) with two REAL ranks on one
GPU, compared with the oracle (VERDICT r01 "Next round" 1(d)).

Two processes share cuda:0 and a gloo process group.  Each builds its
destination-row shard (global source ids), and bench.Step runs the whole step
-- copy_u-sum F512, u_dot_v H1 F512, the GAT chain (u_dot_v H8 D32 -> edge
softmax -> u_mul_e-sum), copy_u-max F128 + args, mlp-max + args -- through
the C ABI, with the source-feature all-gather done by a test-only host shim
of `Comm.allgather_rows`' signature (the gloo stand-in for NCCL, which needs
one GPU per rank).  Every rank checks ITS rows against the oracle on the
all-gathered inputs: bit-exact where the bar says so (max values, argmax),
1e-4 * sum|terms| elsewhere.  The e2e pipelined form of the step
(enqueue_pipelined: host copies, row halves) must reproduce the plain step
bit for bit on every rank."""
import os
import socket
import traceback

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
TOL = 1e-4


class HostAllGather:
    """allgather_rows(offsets, X_local, X_full, stream) over gloo: every rank's
    row block lands in X_full at its offset (what fg_allgather_rows does with
    NCCL broadcasts), ordered after the work already on `stream`."""

    def __init__(self, rank, world):
        self.rank, self.world = rank, world

    def allgather_rows(self, offsets, X_local, X_full, stream=None):
        (stream or torch.cuda.current_stream()).synchronize()
        blocks = []
        for r in range(self.world):
            lo, hi = int(offsets[r]), int(offsets[r + 1])
            b = X_local.detach().cpu().clone() if r == self.rank else torch.empty((hi - lo,) + tuple(X_full.shape[1:]))
            dist.broadcast(b, src=r)
            blocks.append(b)
        with torch.cuda.stream(stream or torch.cuda.current_stream()):
            X_full.copy_(torch.cat(blocks).to(X_full.device))
        return X_full


def _check(gpu, ref, ab, what):
    gpu = np.asarray(gpu, np.float64)
    bad = np.abs(gpu - ref) > TOL * ab
    assert not bad.any(), f"{what}: {int(bad.sum())} elements out of tolerance"


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import bench
        import gen
        import oracle
        from paper_2008_11359_b200.shard import make_shard
        g = gen.random_graph(3000, 150000, 41, sigma=1.6, n_empty=30)
        host = bench.make_inputs(g)
        sh = make_shard(g.row_ptr, g.col_idx, rank, world)
        st = torch.cuda.Stream()
        S = bench.Step(g, sh, host, HostAllGather(rank, world), st)
        # the shard's own rows start with stale copies of the other ranks' features:
        # only the all-gather can make them right
        for k in S.X:
            S.X[k].zero_()
            S.X[k][S.lo:S.lo + S.nl].copy_(torch.from_numpy(host[k][S.lo:S.lo + S.nl]))
        with torch.cuda.stream(st):
            S.enqueue()
        torch.cuda.synchronize()
        rows = np.arange(sh.lo, sh.hi)
        rp, ci = g.row_ptr, g.col_idx
        X512, X256, X128, X8, W = host["X512"], host["X256"], host["X128"], host["X8"], host["W"]
        ref, ab, _, _ = oracle.spmm(rp, ci, "copy_u", "sum", X512, rows=rows)
        _check(S.out512.cpu().numpy(), ref, ab, "copy_u-sum F512")
        pos = oracle.edge_positions(rp, rows)
        rs, rab = oracle.sddmm(rp, ci, X512, rows=rows)
        _check(S.s1.cpu().numpy(), rs, rab, "u_dot_v H1 F512")
        # GAT chain end to end against the fused-layer definition (X256 is scaled
        # to keep the scores small, so the chain's fp32 scores do not amplify)
        rg, rgb = oracle.gat(rp[sh.lo:sh.hi + 1] - rp[sh.lo], ci[pos], X256, X256[sh.lo:sh.hi], H=bench.H_GAT)
        _check(S.o256.cpu().numpy(), rg, rgb, "GAT chain")
        mx, _, rau, rae = oracle.spmm(rp, ci, "copy_u", "max", X128, rows=rows)
        assert np.array_equal(S.o128.cpu().numpy().astype(np.float64), mx), "copy_u-max values"
        assert np.array_equal(S.au128.cpu().numpy(), rau), "copy_u-max arg_u"
        # the shard's local graph numbers its edges from its first edge (identity ids):
        # global edge id = local id + the shard's first CSR position
        ae = S.ae128.cpu().numpy().astype(np.int64)
        assert np.array_equal(np.where(ae >= 0, ae + sh.edge_lo, -1), rae), "copy_u-max arg_e"
        mref, mab, _, _ = oracle.spmm(rp, ci, "mlp", "max", X8, W=W, rows=rows)
        _check(S.omlp.cpu().numpy(), mref, mab, "mlp-max")
        au = S.aumlp.cpu().numpy()
        X64, W64 = X8.astype(np.float64), W.astype(np.float64)
        for i in range(0, sh.hi - sh.lo, 17):
            v = sh.lo + i
            if rp[v + 1] == rp[v]:
                assert (au[i] == -1).all()
                continue
            msg = np.maximum(((X64[au[i]] + X64[v][None, :]) * W64.T).sum(1), 0.0)
            assert (np.abs(msg - mref[i]) <= TOL * mab[i] + 1e-30).all(), "mlp argmax not valid"
        # the e2e (pipelined) form reproduces the plain step bit for bit
        outs = [o.clone() for o in S.outputs()]
        ins = {k: torch.from_numpy(np.ascontiguousarray(host[k][S.lo:S.lo + S.nl])).pin_memory()
               for k in ("X512", "X256", "X128", "X8")}
        w_h = torch.from_numpy(host["W"]).pin_memory()
        outs_h = {id(o): torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in S.outputs()}
        for o in S.outputs():
            o.zero_()
        h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
        with torch.cuda.stream(st):
            S.enqueue_pipelined(ins, w_h, outs_h, h2d, d2h)
            st.wait_stream(d2h)
        torch.cuda.synchronize()
        for o, ref_o in zip(S.outputs(), outs):
            assert torch.equal(outs_h[id(o)], ref_o.cpu()), "pipelined step differs"
        q.put((rank, "ok"))
    except Exception:  # noqa: BLE001
        q.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_step_two_ranks_one_gpu(cuda_ok):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert res[r] == "ok", f"rank {r}:\n{res[r]}"
    assert all(p.exitcode == 0 for p in procs)
