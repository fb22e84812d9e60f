#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for the FeatGraph hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1: dst-row sharded)

Workload (BASELINE.json metric "gSpMM/gSDDMM ms/op & HBM GB/s vs ~8 TB/s, feat
32-512"; north-star target graph): the reddit-shaped synthetic graph
(232,965 vertices, 114,615,892 edges, lognormal in-degrees, Chung-Lu sources;
DESIGN.md "Input recipe").  One STEP = one pass of every SURVEY §8(a) row over
that graph, fp32:
    a1  gSpMM copy_u-sum   F=512              (GCN aggregation, Table tab:gpu-kernel(a))
    a4  gSDDMM u_dot_v     H=1, F=512         (dot-product attention, tab:gpu-kernel(c))
    a4  gSDDMM u_dot_v     H=8, D=32          (GAT scores, BASELINE configs[2])
    a5  edge softmax       H=8                (in place)
    a2  gSpMM u_mul_e-sum  H=8, D=32          (GAT aggregation)
    a1  gSpMM copy_u-max   F=128 + arg_u/arg_e
    a3  gSpMM mlp-max      d1=8, d2=128 + args (MLP aggregation, tab:gpu-kernel(b))
    a6  (N > 1) NCCL all-gather of every source-feature tensor (row shards)
a0 (fg_graph_create) is per-topology preprocessing, amortised and
outside the step.

value = algorithmic bytes of the step (SURVEY §8(d) gather model, summed over
ops, whole graph) / device time per step (CUDA events on the launching stream,
max over ranks), in GB/s.  L2 is flushed (256 MB write) before every timed
step, outside the timed events.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GRAPH = "reddit"
F_GCN, F_DOT, H_GAT, D_GAT, F_MAX, D1, D2 = 512, 512, 8, 32, 128, 8, 128
OPS = ["spmm_copy_u_sum_F512", "sddmm_u_dot_v_H1_F512", "sddmm_u_dot_v_H8_D32", "edge_softmax_H8",
       "spmm_u_mul_e_sum_H8_D32", "spmm_copy_u_max_F128_args", "spmm_mlp_max_d8_d128_args"]


def metric_name() -> str:
    try:
        return json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
    except Exception:
        return "gSpMM/gSDDMM ms/op & HBM GB/s vs ~8 TB/s, feat 32-512, at 1/2/4/8 B200"


def run_backward(S, timed, sync_all) -> dict:
    """Row f1 at full size (reddit-shaped, N = 1): the gradients of the step's
    ops through the gradient duality, each timed like the extras
    (CUDA events, L2 flushed, mean of k).  Bytes: the gather model of the
    forward op each gradient runs as (dX = a gSpMM over the transposed handle,
    dE / dY = a gSDDMM / gSpMM over the graph; the max gradient reads the
    forward's arg_u once per (edge, feature) it tests)."""
    import torch
    fgp, st, G, X, n, m = S.fgp, S.stream, S.G, S.X, S.nl, S.m
    GT = G.transpose(stream=st)
    sync_all()
    idx = 8 * (n + 1) + 4 * m
    r = {}

    def put(name, ms, b):
        r[name] = {"ms": round(ms, 4), "gbs": round(b / (ms * 1e-3) / 1e9, 1)}

    # copy_u-sum F=512: dX = spmm(gT, dOut)
    dout = S.out512
    put("spmm_copy_u_sum_F512_dX", timed(lambda: fgp.spmm_backward(G, GT, "copy_u", "sum", dout, stream=st)),
        idx + 4 * m * F_GCN + 4 * n * F_GCN)
    # u_mul_e-sum H=8 D=32: dX over gT (weighted by E) and dE = sddmm(g, X, dOut)
    d256 = S.o256
    put("spmm_u_mul_e_sum_H8_D32_dX_dE", timed(lambda: fgp.spmm_backward(
        G, GT, "u_mul_e", "sum", d256, H=H_GAT, X=X["X256"], E=S.s8, want_dE=True, stream=st)),
        2 * idx + 2 * 4 * m * H_GAT * D_GAT + 2 * 4 * m * H_GAT + 2 * 4 * n * H_GAT * D_GAT)
    # copy_u-max F=128: dX masked by the forward's arg_u (gathers dOut and arg_u per edge)
    put("spmm_copy_u_max_F128_dX", timed(lambda: fgp.spmm_backward(
        G, GT, "copy_u", "max", S.o128, X=X["X128"], arg_u=S.au128, stream=st)),
        idx + 2 * 4 * m * F_MAX + 4 * n * F_MAX)
    # u_dot_v H=8 D=32: dX = spmm_{u_mul_e}(gT, Y, dS), dY = spmm_{u_mul_e}(g, X, dS)
    put("sddmm_u_dot_v_H8_D32_dX_dY", timed(lambda: fgp.sddmm_backward(
        G, GT, X["X256"], S.ydst("X256"), S.s8, H=H_GAT, stream=st)),
        2 * (idx + 4 * m * H_GAT * D_GAT + 4 * m * H_GAT + 4 * n * H_GAT * D_GAT))
    # edge softmax H=8: ds = alpha * (dalpha - sum_row alpha * dalpha)
    # (alpha = dalpha = the step's alpha: the timing does not depend on the values)
    put("edge_softmax_H8_ds", timed(lambda: fgp.edge_softmax_backward(G, S.s8, S.s8, H=H_GAT, stream=st)),
        8 * (n + 1) + 3 * 4 * m * H_GAT)
    del GT
    torch.cuda.empty_cache()
    return r


def op_bytes(n_rows: int, m: int) -> dict:
    """Algorithmic bytes per op (SURVEY §8(d) gather model; row_ptr is int64):
    index arrays + per-edge source-row gathers + per-row reads/writes."""
    idx = 8 * (n_rows + 1) + 4 * m
    return {
        "spmm_copy_u_sum_F512": idx + 4 * m * F_GCN + 4 * n_rows * F_GCN,
        "sddmm_u_dot_v_H1_F512": idx + 4 * m * F_DOT + 4 * n_rows * F_DOT + 4 * m,
        "sddmm_u_dot_v_H8_D32": idx + 4 * m * H_GAT * D_GAT + 4 * n_rows * H_GAT * D_GAT + 4 * m * H_GAT,
        "edge_softmax_H8": 8 * (n_rows + 1) + 2 * 4 * m * H_GAT,
        "spmm_u_mul_e_sum_H8_D32": idx + 4 * m * H_GAT * D_GAT + 4 * m * H_GAT + 4 * n_rows * H_GAT * D_GAT,
        "spmm_copy_u_max_F128_args": idx + 4 * m * F_MAX + 3 * 4 * n_rows * F_MAX,
        "spmm_mlp_max_d8_d128_args": idx + 4 * m * D1 + 4 * n_rows * D1 + 4 * D1 * D2 + 3 * 4 * n_rows * D2,
    }


def mlp_flops(m: int) -> int:
    return 2 * m * D1 * D2


# ----------------------------------------------------------------- inputs (host, seeded)
def make_inputs(g):
    import gen
    s = gen.feature_seed(GRAPH)
    n = g.n_dst
    return {
        "X512": gen.features((n, F_GCN), s, 0),
        "X256": gen.features((n, H_GAT * D_GAT), s, 1) * np.float32(0.25),
        "X128": gen.features((n, F_MAX), s, 2),
        "X8": gen.features((n, D1), s, 3),
        "W": gen.features((D1, D2), s, 4, gen.SCALED, scale=1 / np.sqrt(D1)),
    }


# ----------------------------------------------------------------- clocks sampler
class Clocks:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, dev_id: str):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", dev_id, "--query-gpu=" + ",".join(self.FIELDS), "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self) -> dict | None:
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


def gpu_id_for_smi(local_rank: int) -> str:
    import torch
    try:
        u = str(torch.cuda.get_device_properties(local_rank).uuid)
        if u and u != "None":
            return u if u.startswith("GPU-") else "GPU-" + u
    except Exception:
        pass
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        return vis.split(",")[local_rank]
    return str(local_rank)


def l2_gather_ceiling(torch, buf) -> dict | None:
    """The L2 gather ceiling of this GPU, measured live (libfgprobe.so,
    paper_2008_11359_b200/probe/l2_probe.cu): random whole-row reads of an
    L2-resident 64 MiB X with the kernels' lane mapping, no arithmetic.  The
    roofline denominator for the gather kernels whose source rows mostly hit L2."""
    import ctypes
    path = os.path.join(ROOT, "paper_2008_11359_b200", "lib", "libfgprobe.so")
    if not os.path.exists(path):
        return None
    L = ctypes.CDLL(path)
    L.fgprobe_l2.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_double)]
    out = (ctypes.c_double * 5)()
    torch.cuda.synchronize()
    rc = L.fgprobe_l2(ctypes.c_void_p(buf.data_ptr()), buf.numel() * buf.element_size(), out)
    if rc != 0:
        return None
    return {"gather_2k_rows": round(out[0], 1), "gather_512b_rows": round(out[1], 1),
            "gather_128b_rows": round(out[2], 1), "stream": round(out[3], 1), "gather_best": round(out[4], 1)}


class L2Flush:
    """Write a 256 MB buffer (2x the 126 MB L2), then read it back: afterwards the
    L2 holds only clean flush lines, so no write-back of the flush itself lands
    inside the next timed region."""

    def __init__(self, torch):
        self.torch = torch
        self.buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
        self.sink = torch.empty((), dtype=torch.float32, device="cuda")

    def fill_(self, v: float):
        self.buf.fill_(v)
        self.torch.sum(self.buf, 0, out=self.sink)


# ----------------------------------------------------------------- the GPU step
class Step:
    """Device-resident state of one rank and the enqueue of one hot-path step."""

    def __init__(self, g, shard, host, comm, stream):
        import torch
        import paper_2008_11359_b200 as fgp
        from paper_2008_11359_b200.shard import make_shard as make_shard_fn
        self.fgp, self.torch = fgp, torch
        self.shard, self.comm, self.stream = shard, comm, stream
        self.n = g.n_dst
        nl = shard.n_local if shard else g.n_dst
        self.nl = nl
        lo = shard.lo if shard else 0
        dev = torch.device("cuda")
        rp = shard.row_ptr if shard else g.row_ptr
        ci = shard.col_idx if shard else g.col_idx
        self.rp_d = torch.from_numpy(rp).to(dev)
        self.ci_d = torch.from_numpy(ci).to(dev)
        self.G = fgp.Graph(self.rp_d, self.ci_d, n_src=g.n_src, validate=True)
        self.prepare(self.G, g.nnz)
        self.m = int(rp[-1])
        self.lo = lo
        # full-size source feature buffers (the all-gather target when sharded)
        self.X = {k: torch.from_numpy(host[k]).to(dev) for k in ("X512", "X256", "X128", "X8")}
        self.W = torch.from_numpy(host["W"]).to(dev)
        f = lambda *s: torch.empty(*s, device=dev)  # noqa: E731
        i = lambda *s: torch.empty(*s, dtype=torch.int32, device=dev)  # noqa: E731
        self.out512 = f(nl, F_GCN)
        self.s1 = f(self.m, 1)
        self.s8 = f(self.m, H_GAT)
        self.o256 = f(nl, H_GAT * D_GAT)
        self.o128, self.au128, self.ae128 = f(nl, F_MAX), i(nl, F_MAX), i(nl, F_MAX)
        self.omlp, self.aumlp, self.aemlp = f(nl, D2), i(nl, D2), i(nl, D2)
        self.ev = None
        # N > 1: the source-feature all-gathers run on their own stream, in the
        # order the ops consume them, overlapped with the ops on the earlier tensors
        self.comm_stream = torch.cuda.Stream() if comm is not None else None
        # e2e leg: the last op (GAT aggregation) runs on two row halves of this
        # rank's graph (two fg_graph handles over contiguous row ranges, global
        # source ids) so the first half's result ships while the second computes
        # (the X512 ops on halves, the final GAT aggregation on quarters: its last
        # piece's D2H is the e2e tail)
        self.halves = self.row_pieces(fgp, torch, dev, g, rp, ci, make_shard_fn, 2)
        self.quarters = self.row_pieces(fgp, torch, dev, g, rp, ci, make_shard_fn, 4)

    def row_pieces(self, fgp, torch, dev, g, rp, ci, make_shard_fn, k):
        """k nnz-balanced contiguous row ranges of this rank's graph as fg_graph
        handles (global source ids): [(handle, row_lo, row_hi, edge_lo, edge_hi)].
        Each split row is moved to the nearest row whose first edge is a multiple
        of 4 (the per-edge H=1 scores s1[e0:e1] must stay 16-byte aligned)."""
        offs = [0]
        for q in range(1, k):
            mid = int(np.searchsorted(rp, rp[-1] * q // k))
            cand = [r for r in range(max(1, mid - 64), min(len(rp) - 1, mid + 64)) if rp[r] % 4 == 0]
            offs.append(max(offs[-1], min(cand, key=lambda r: abs(r - mid)) if cand else 0))
        offs.append(len(rp) - 1)
        offs = np.array(offs, np.int64)
        pieces = []
        for r in range(k):
            h = make_shard_fn(rp, ci, r, k, offsets=offs)
            Gh = fgp.Graph(torch.from_numpy(h.row_ptr).to(dev), torch.from_numpy(h.col_idx).to(dev), n_src=g.n_src)
            self.prepare(Gh, g.nnz)
            pieces.append((Gh, h.lo, h.hi, h.edge_lo, h.edge_lo + h.nnz))
        return pieces

    @staticmethod
    def prepare(G, nnz_total):
        """Per-topology setup outside the timed region: the source-segment tables of
        the gathered widths (fp32 F = 512 / 256 and their bf16 storage), and the
        whole graph's edge count for the CTA-per-row threshold (so shards and row
        halves split rows exactly as the unsharded op)."""
        G.tune("balance_nnz", nnz_total)
        for row_bytes in (F_DOT * 4, H_GAT * D_GAT * 4, F_DOT * 2, H_GAT * D_GAT * 2):
            G.prepare(row_bytes)

    def ydst(self, k):
        return self.X[k][self.lo:self.lo + self.nl]

    GATHER_ORDER = ("X512", "X256", "X128", "X8")

    def allgather_async(self) -> dict:
        """Enqueue the all-gather of every source-feature tensor on comm_stream
        (after everything already on the compute stream: the previous step's ops
        still read the non-local rows); returns key -> event marking its arrival."""
        if self.comm is None:
            return {}
        cs, torch = self.comm_stream, self.torch
        cs.wait_stream(self.stream)
        done = {}
        for k in self.GATHER_ORDER:
            x = self.X[k]
            self.comm.allgather_rows(self.shard.offsets, x[self.lo:self.lo + self.nl], x, stream=cs)
            done[k] = torch.cuda.Event()
            done[k].record(cs)
        return done

    def enqueue(self, events=None):
        """All ops of one step on self.stream; events[i] recorded before op i (and at the end)."""
        fgp, st = self.fgp, self.stream
        rec = (lambda i: events[i].record(st)) if events is not None else (lambda i: None)
        G, X = self.G, self.X
        rec(0)
        arrived = self.allgather_async()

        def need(k):   # the compute stream waits for tensor k's all-gather (N > 1)
            if k in arrived:
                st.wait_event(arrived[k])

        need("X512")
        rec(1)
        fgp.spmm(G, "copy_u", "sum", X["X512"], out=self.out512, stream=st)
        rec(2)
        fgp.sddmm(G, X["X512"], self.ydst("X512"), H=1, out=self.s1, stream=st)
        rec(3)
        need("X256")
        fgp.sddmm(G, X["X256"], self.ydst("X256"), H=H_GAT, out=self.s8, stream=st)
        rec(4)
        fgp.edge_softmax(G, self.s8, H=H_GAT, out=self.s8, stream=st)
        rec(5)
        fgp.spmm(G, "u_mul_e", "sum", X["X256"], H=H_GAT, E=self.s8, out=self.o256, stream=st)
        rec(6)
        need("X128")
        fgp.spmm(G, "copy_u", "max", X["X128"], out=self.o128, arg_u=self.au128, arg_e=self.ae128, stream=st)
        rec(7)
        need("X8")
        fgp.spmm(G, "mlp", "max", X["X8"], W=self.W, X_dst=self.ydst("X8"), out=self.omlp, arg_u=self.aumlp,
                 arg_e=self.aemlp, stream=st)
        rec(8)

    LAUNCHES_PER_STEP = 7   # libfg kernels per step: one per fg_* call

    def enqueue_pipelined(self, ins_h, w_h, outs_h, h2d, d2h):
        """The same step for the end-to-end leg, with the host copies overlapped:
        H2D of each input on stream h2d (in the order the ops need them), each op
        on self.stream as soon as its input has arrived (smallest inputs first,
        the smallest result last), and the D2H
        of each op's results on stream d2h as soon as that op is done.  Callers
        make h2d / d2h wait on the start event and self.stream wait on d2h at
        the end."""
        fgp, st, torch = self.fgp, self.stream, self.torch
        G, X, lo, nl = self.G, self.X, self.lo, self.nl
        arrived = {}
        with torch.cuda.stream(h2d):
            for key in ("X8", "X128", "X256", "X512"):   # in the order the ops below first need them
                X[key][lo:lo + nl].copy_(ins_h[key], non_blocking=True)
                if key == "X8":
                    self.W.copy_(w_h, non_blocking=True)
                arrived[key] = torch.cuda.Event()
                arrived[key].record(h2d)

        def ready(key):
            st.wait_event(arrived[key])
            if self.comm is not None:
                self.comm.allgather_rows(self.shard.offsets, X[key][lo:lo + nl], X[key], stream=st)

        def ship(outs, rows=None):
            done = torch.cuda.Event()
            done.record(st)
            d2h.wait_event(done)
            with torch.cuda.stream(d2h):
                for o in outs:
                    if rows is None:
                        outs_h[id(o)].copy_(o, non_blocking=True)
                    else:
                        outs_h[id(o)][rows[0]:rows[1]].copy_(o[rows[0]:rows[1]], non_blocking=True)

        # op order: the smallest input first (X8, 7.5 MB), and the GAT scores +
        # softmax (X256) before copy_u-sum so that X512's 477 MB copy is hidden
        # behind them; the GAT aggregation last -- its n x 256 result is the
        # smallest D2H tail
        ready("X8")
        fgp.spmm(G, "mlp", "max", X["X8"], W=self.W, X_dst=self.ydst("X8"), out=self.omlp, arg_u=self.aumlp,
                 arg_e=self.aemlp, stream=st)
        ship([self.omlp, self.aumlp, self.aemlp])
        ready("X128")
        fgp.spmm(G, "copy_u", "max", X["X128"], out=self.o128, arg_u=self.au128, arg_e=self.ae128, stream=st)
        ship([self.o128, self.au128, self.ae128])
        ready("X256")
        fgp.sddmm(G, X["X256"], self.ydst("X256"), H=H_GAT, out=self.s8, stream=st)
        fgp.edge_softmax(G, self.s8, H=H_GAT, out=self.s8, stream=st)
        ready("X512")
        # the two X512 ops on the row halves too: each half's result ships while
        # the next half computes (the D2H stream is the e2e tail's bottleneck)
        for Gh, rlo, rhi, elo, ehi in self.halves:
            fgp.spmm(Gh, "copy_u", "sum", X["X512"], out=self.out512[rlo:rhi], stream=st)
            ship([self.out512], rows=(rlo, rhi))
        for Gh, rlo, rhi, elo, ehi in self.halves:
            fgp.sddmm(Gh, X["X512"], self.ydst("X512")[rlo:rhi], H=1, out=self.s1[elo:ehi], stream=st)
            ship([self.s1], rows=(elo, ehi))
        for Gh, rlo, rhi, elo, ehi in self.quarters:   # each quarter's D2H overlaps the next
            fgp.spmm(Gh, "u_mul_e", "sum", X["X256"], H=H_GAT, E=self.s8[elo:ehi], out=self.o256[rlo:rhi], stream=st)
            ship([self.o256], rows=(rlo, rhi))

    def outputs(self):
        return [self.out512, self.s1, self.o256, self.o128, self.au128, self.ae128, self.omlp, self.aumlp,
                self.aemlp]


# ----------------------------------------------------------------- CPU oracle leg
def oracle_sample_step(g, host, rows):
    """Run every op of the step with the fp64 oracle on the sub-graph of `rows`
    (their in-edges, global source ids).  Returns (seconds, bytes, threads)."""
    import oracle
    rows = np.sort(np.asarray(rows, np.int64))
    deg = g.row_ptr[rows + 1] - g.row_ptr[rows]
    rp = np.zeros(rows.size + 1, np.int64)
    np.cumsum(deg, out=rp[1:])
    pos = oracle.edge_positions(g.row_ptr, rows)
    ci = g.col_idx[pos]
    X512, X256, X128, X8, W = host["X512"], host["X256"], host["X128"], host["X8"], host["W"]
    t0 = time.perf_counter()
    oracle.spmm(rp, ci, "copy_u", "sum", X512)
    oracle.sddmm(rp, ci, X512, X512[rows], H=1)
    s8, _ = oracle.sddmm(rp, ci, X256, X256[rows], H=H_GAT)
    a8 = oracle.edge_softmax(rp, s8.astype(np.float32), H=H_GAT)
    oracle.spmm(rp, ci, "u_mul_e", "sum", X256, H=H_GAT, E=a8.astype(np.float32))
    oracle.spmm(rp, ci, "copy_u", "max", X128)
    oracle.spmm(rp, ci, "mlp", "max", X8, W=W, X_dst=X8[rows])
    dt = time.perf_counter() - t0
    b = sum(op_bytes(rows.size, int(rp[-1])).values())
    return dt, b, int(rp[-1])


def sample_rows(g, edge_budget: int, seed: int = 11) -> np.ndarray:
    import gen
    perm = gen.permutation(g.n_dst, seed, 31)
    deg = np.diff(g.row_ptr)[perm]
    k = int(np.searchsorted(np.cumsum(deg), edge_budget)) + 1
    return perm[:max(1, min(k, g.n_dst))]


def cpu_threads() -> int:
    try:
        return int(os.environ.get("OMP_NUM_THREADS") or len(os.sched_getaffinity(0)))
    except Exception:
        return os.cpu_count() or 1


def calibrate_sample(g, host, target_s: float):
    """Grow a seeded row sample until one oracle step takes ~target_s.  Returns
    (rows, seconds, bytes, edges) of the LAST (reported) measurement."""
    budget = 20000
    while True:
        rows = sample_rows(g, budget)
        dt, b, me = oracle_sample_step(g, host, rows)
        if dt >= 0.5 * target_s or budget >= g.nnz:
            return rows, dt, b, me
        budget = min(g.nnz, int(budget * min(8.0, max(1.5, 0.9 * target_s / max(dt, 1e-3)))))


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_c2_single_thread() -> dict:
    """The analogue of Table tab:cpu-kernel's single-thread protocol:
    the fp64 oracle's copy_u-sum at F = 32 on a seeded row sample of the
    proteins-shaped graph, ONE thread (a fresh process with OMP_NUM_THREADS=1).
    Context only: the oracle is a correctness reference, not a tuned kernel."""
    code = ("import sys, time, json; sys.path.insert(0, %r); import numpy as np, gen, oracle, bench;"
            "g = gen.make_graph('proteins'); rows = bench.sample_rows(g, 2_000_000);"
            "rows = np.sort(rows); X = gen.features((g.n_src, 32), gen.feature_seed('proteins'), 0);"
            "deg = g.row_ptr[rows + 1] - g.row_ptr[rows]; rp = np.zeros(rows.size + 1, np.int64);"
            "np.cumsum(deg, out=rp[1:]); ci = g.col_idx[oracle.edge_positions(g.row_ptr, rows)];"
            "oracle.spmm(rp[:2], ci[:rp[1]], 'copy_u', 'sum', X);"
            "t = time.perf_counter(); oracle.spmm(rp, ci, 'copy_u', 'sum', X); dt = time.perf_counter() - t;"
            "print(json.dumps({'rows': int(rows.size), 'edges': int(rp[-1]), 'seconds': dt}))") % ROOT
    env = dict(os.environ, OMP_NUM_THREADS="1")
    try:
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        d = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        return {"error": str(e)[:200]}
    full_s = d["seconds"] * 79122504 / max(d["edges"], 1)
    return {"op": "copy_u-sum F=32 (proteins-shaped)", "threads": 1, "sample_rows": d["rows"],
            "sample_edges": d["edges"], "sample_s": round(d["seconds"], 3),
            "extrapolated_full_graph_ms": round(full_s * 1e3, 1)}


def cpu_baseline(g, host, target_s: float = 12.0) -> dict:
    rows, dt, b, me = calibrate_sample(g, host, target_s)
    return {"value": b / dt / 1e9, "unit": "GB/s", "cores": cpu_threads(), "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"all 7 ops of the step on {rows.size} seeded-random destination rows "
                      f"({me} in-edges, {me / g.nnz:.2%} of the graph), fp64 C oracle, OpenMP over rows; "
                      f"{dt:.1f} s", "seconds": dt,
            "single_thread_c2": oracle_c2_single_thread()}


# ----------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--uniform-sources", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU harness: start the ranks (gloo), report them, skip all GPU work")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `bench.py --gpus N` without a launcher: re-exec under torch.distributed.run,
        # one rank per GPU (the driver's own launch form), NCCL init logged
        return self_launch(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"bench.py: WORLD_SIZE={world} overrides --gpus {args.gpus}", file=sys.stderr)
    if args.dry_run:
        return dry_run(args, world, rank)
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import torch.distributed as dist
    import gen
    import paper_2008_11359_b200 as fgp
    from paper_2008_11359_b200.shard import make_shard

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    g = gen.make_graph(GRAPH, uniform_sources=args.uniform_sources)
    host = make_inputs(g)
    comm, shard = None, None
    if world > 1:
        shard = make_shard(g.row_ptr, g.col_idx, rank, world)
        uid = [fgp.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = fgp.Comm(uid[0], world, rank)
    stream = torch.cuda.Stream()
    S = Step(g, shard, host, comm, stream)
    S.total_bytes = sum(op_bytes(g.n_dst, g.nnz).values())
    flush = L2Flush(torch)

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            flush.fill_(1.0)
            S.enqueue()
    sync_all()
    nev = 9
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nev)] for _ in range(args.steps)]
    clocks = Clocks(gpu_id_for_smi(local_rank)) if rank == 0 else None
    time.sleep(0.3 if rank == 0 else 0)
    sync_all()
    with torch.cuda.stream(stream):
        for k in range(args.steps):
            flush.fill_(float(k))        # L2 flush outside the timed events
            S.enqueue(evs[k])
    sync_all()
    clk = clocks.stop() if clocks else None
    step_ms = np.array([evs[k][0].elapsed_time(evs[k][8]) for k in range(args.steps)])
    op_ms = {OPS[i]: float(np.mean([evs[k][i + 1].elapsed_time(evs[k][i + 2]) for k in range(args.steps)]))
             for i in range(7)}
    ag_ms = float(np.mean([evs[k][0].elapsed_time(evs[k][1]) for k in range(args.steps)]))
    ms = float(step_ms.mean())
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # the paper's protocol: the same step with L2 left warm between runs
    warm_ms = timed_steps(S, args.steps, None, torch)
    if world > 1:
        t = torch.tensor([warm_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        warm_ms = float(t.item())

    # next rows and the other BASELINE configs, timed beside the step (not part of it)
    extras = None if args.no_extras else run_extras(S, args, sync_all, flush, world)

    # end-to-end through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(S, host, args, world, sync_all, flush)

    l2peak = l2_gather_ceiling(torch, flush.buf) if rank == 0 else None
    total_bytes = sum(op_bytes(g.n_dst, g.nnz).values())
    local_bytes = op_bytes(S.nl, S.m)
    ob_full = op_bytes(g.n_dst, g.nnz)
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(g, host)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    sm_mhz = (clk or {}).get("sm_mhz") or float(peaks.get("sm_max_mhz", 1965.0))
    # dominant kernel = the HBM/L2-bound op with the largest share of the step
    dom = max((k for k in op_ms if k != "spmm_mlp_max_d8_d128_args"), key=lambda k: op_ms[k])
    roof = roofline(dom, op_ms[dom], local_bytes[dom], op_ms, hbm_peak, l2peak, world,
                    "uniform" if args.uniform_sources else "default")
    mlp_ms = op_ms["spmm_mlp_max_d8_d128_args"]
    line = {
        "metric": metric_name(),
        "value": total_bytes / (ms * 1e-3) / 1e9,
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": {
            "workload": "reddit-shaped synthetic graph (232,965 v, 114,615,892 e; lognormal sigma=1.2, "
                        "Chung-Lu sources" + (", UNIFORM sources" if args.uniform_sources else "") +
                        "): copy_u-sum F512, u_dot_v H1 F512, GAT (u_dot_v H8D32 -> edge_softmax -> "
                        "u_mul_e-sum), copy_u-max F128+argmax, mlp-max d1=8 d2=128+argmax",
            "graph": GRAPH, "n": g.n_dst, "nnz": g.nnz,
            "parallelism": (f"dst-row shards x{world} + NCCL all-gather of X (own stream, overlapped with the "
                            "ops on earlier tensors; allgather_ms = the exposed wait for X512)")
            if world > 1 else "single GPU",
            "l2": "flushed before every timed step, outside the events: 256 MB write (2x the L2) then a "
                  "read of it, so the flush's dirty lines are written back before the step starts "
                  "(warm_l2_ms_per_step: the paper's warm protocol, P:607)",
            "bytes_per_step": total_bytes,
            "value_bytes": "gather model (SURVEY 8(d)): every per-edge source-row read counted at full width; "
                           "L2 serves most of them, so value is an effective rate, not a physical HBM rate "
                           "(roofline.dram_gbs is the physical one)",
        },
        "warm_l2_ms_per_step": round(warm_ms, 4),
        "ops_ms": {k: round(v, 4) for k, v in op_ms.items()},
        "ops_gbs": {k: round(ob_full[k] / world / (op_ms[k] * 1e-3) / 1e9, 1) for k in OPS} if world == 1 else
        {k: round(local_bytes[k] / (op_ms[k] * 1e-3) / 1e9, 1) for k in OPS},
        "allgather_ms": round(ag_ms, 4) if world > 1 else 0.0,
        "comm": ({"backend": "nccl", "nranks": S.comm.nranks_nccl()} if world > 1 else None),
        "mlp_tflops": round(mlp_flops(S.m) / (mlp_ms * 1e-3) / 1e12, 2),
        "mlp_roofline": mlp_roofline(S.m, mlp_ms, sm_mhz),
        "roofline": roof,
        "ops_physical": ops_physical(op_ms, hbm_peak, world, "uniform" if args.uniform_sources else "default"),
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": Step.LAUNCHES_PER_STEP * args.steps,
        "clocks": clk,
        "extras": extras,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def self_launch(n: int) -> int:
    """Re-exec this command under torch.distributed.run with n ranks on
    127.0.0.1 (one process per GPU); NCCL's communicator init is logged
    (NCCL_DEBUG=INFO, subsystem INIT) unless the caller set NCCL_DEBUG."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    print("bench.py: self-launch: " + " ".join(cmd), file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


def dry_run(args, world: int, rank: int) -> int:
    """Launch check without a GPU: the ranks meet over gloo, agree on the world
    size and the row shards of a small graph, and rank 0 prints the JSON line."""
    import torch.distributed as dist
    import gen
    from paper_2008_11359_b200.shard import make_shard
    if world > 1:
        dist.init_process_group("gloo")
    g = gen.random_graph(2000, 40000, 5)
    sh = make_shard(g.row_ptr, g.col_idx, rank, world)
    print(f"bench.py dry-run: rank {rank}/{world} rows [{sh.lo}, {sh.hi}) nnz {sh.nnz}", file=sys.stderr, flush=True)
    ranks = [None] * world
    if world > 1:
        dist.all_gather_object(ranks, (rank, sh.lo, sh.hi, sh.nnz))
    else:
        ranks = [(rank, sh.lo, sh.hi, sh.nnz)]
    if rank == 0:
        print(json.dumps({"metric": metric_name(), "dry_run": True, "n_gpus": world,
                          "ranks": [list(r) for r in ranks], "nnz_total": int(sum(r[3] for r in ranks))}),
              flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def timed_steps(S, k_steps: int, flush, torch) -> float:
    """Mean device ms of k_steps whole steps on S.stream (after one untimed step);
    flush=None keeps L2 warm between steps (the paper's protocol)."""
    st = S.stream
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k_steps + 1)]
    with torch.cuda.stream(st):
        for k in range(k_steps + 1):
            if flush is not None:
                flush.fill_(float(k))
            evs[k][0].record(st)
            S.enqueue()
            evs[k][1].record(st)
    torch.cuda.synchronize()
    return float(np.mean([evs[k][0].elapsed_time(evs[k][1]) for k in range(1, k_steps + 1)]))


def ncu_record(op: str, variant: str):
    """(record, fresh, stamped_hash) of `op` from profiles/ncu_traffic.json: the
    per-launch ncu figures of the last --set full capture, usable only if that
    capture was taken on the libfg.so this tree builds (same source hash)."""
    from paper_2008_11359_b200.build import source_hash
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        doc = json.load(open(tp))
    except Exception:
        return None, False, None
    h = doc.get("build_hash")
    return doc.get(variant, {}).get(op), h == source_hash(), h


def roofline(dom, dom_ms, dom_bytes, op_ms, hbm_peak, l2peak, world, variant) -> dict:
    """The dominant kernel's roofline line (base contract fields + the physical
    figures).  achieved = gather-model bytes per launch / live event time (the
    contract's algorithmic bytes: per edge 4F bytes of X[u] + index and row
    terms) against the measured HBM copy peak -- an EFFECTIVE rate that L2
    reuse lets exceed 1; dram_* and l2_* are the physical rates: the ncu bytes
    of one launch of this build (profiles/ncu_traffic.json) over the live time."""
    from paper_2008_11359_b200.build import source_hash
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    rec, fresh, stamped = ncu_record(dom, variant)
    r = {"kernel": dom, "share": round(dom_ms / sum(op_ms.values()), 4), "bound": "hbm",
         "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
         "achieved_model": "gather model (effective; not a physical HBM rate -- see dram_gbs / l2_gbs)",
         "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)",
         "traffic": None, "dram_gbs": None, "dram_frac": None, "l2_gbs": None, "l2_frac_of_ncu_peak": None,
         "l2_frac_of_gather_probe": None,
         "ncu": {"build_hash": source_hash(), "capture_hash": stamped, "fresh": bool(fresh and rec)}}
    if rec and fresh and world == 1:
        t = dom_ms * 1e-3
        traffic = rec.get("dram_bytes_per_launch")
        r["traffic"] = traffic
        if traffic:
            r["dram_gbs"] = round(traffic / t / 1e9, 1)
            r["dram_frac"] = round(traffic / t / 1e9 / hbm_peak, 4)
        l2b = rec.get("l2_bytes_per_launch")
        if l2b:
            r["l2_gbs"] = round(l2b / t / 1e9, 1)
            if l2peak:
                r["l2_frac_of_gather_probe"] = round(l2b / t / 1e9 / l2peak["gather_best"], 4)
        pct, nt = rec.get("lts_throughput_pct"), rec.get("ncu_time_s")
        if pct and nt:   # ncu's L2 throughput share, rescaled from the capture's time to this run's
            r["l2_frac_of_ncu_peak"] = round(pct / 100.0 * nt / t, 4)
        r["ncu"]["capture"] = rec.get("capture")
    r["l2_probe"] = l2peak
    return r


def sm_max_mhz() -> float:
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("sm_max_mhz", 1965.0))
    except Exception:
        return 1965.0


def ops_physical(op_ms, hbm_peak, world, variant) -> dict | None:
    """Per op of the step: the physical DRAM and L2 rates (ncu bytes of one
    launch of THIS build, profiles/ncu_traffic.json, over this run's event
    time) -- e.g. the edge softmax, whose traffic must come from HBM, against
    the measured HBM copy peak."""
    if world != 1:
        return None
    res = {}
    for op, ms in op_ms.items():
        rec, fresh, _ = ncu_record(op, variant)
        if not (rec and fresh):
            continue
        t = ms * 1e-3
        d = {"dram_gbs": round(rec["dram_bytes_per_launch"] / t / 1e9, 1),
             "dram_frac": round(rec["dram_bytes_per_launch"] / t / 1e9 / hbm_peak, 4)}
        if rec.get("l2_bytes_per_launch"):
            d["l2_gbs"] = round(rec["l2_bytes_per_launch"] / t / 1e9, 1)
        if rec.get("lts_throughput_pct") and rec.get("ncu_time_s"):
            d["l2_frac_of_ncu_peak"] = round(rec["lts_throughput_pct"] / 100.0 * rec["ncu_time_s"] / t, 4)
        res[op] = d
    return res or None


def mlp_roofline(m: int, ms: float, sm_mhz: float, d2: int = D2, sms: int = 148) -> dict:
    """The tcgen05 MLP kernel against its bound, reading every fp32 accumulator
    element out of TMEM (m x d2 x 4 bytes) at the guide's LDTM throughput of
    64 B/clk/SM (B300_MICROARCH.md "TMEM"; same tcgen05.ld on sm_100a) x SMs x
    the live SM clock; plus the tensor pipe's share (3 tf32 MMAs per product)."""
    tmem_bytes = 4 * m * d2
    peak = 64.0 * sms * sm_mhz * 1e6 / 1e9
    ach = tmem_bytes / (ms * 1e-3) / 1e9
    return {"bound": "tmem-read", "achieved": round(ach, 1), "peak": round(peak, 1), "unit": "GB/s",
            "frac": round(ach / peak, 4),
            "peak_source": f"64 B/clk/SM (guide LDTM throughput) x {sms} SMs x {sm_mhz:.0f} MHz (live median)",
            "algorithmic_tflops": round(2 * m * 8 * d2 / (ms * 1e-3) / 1e12, 2)}


def run_extras(S, args, sync_all, flush, world):
    """Measured beside the step (not part of it):
      f2  fused GAT (u_dot_v -> softmax -> u_mul_e-sum in one pass);
      f4  bf16 feature storage, u_dot_v-then-e_mul;
      a3  MLP ablations on the same reddit inputs (FFMA, bf16 2-split vs 3xTF32);
    and, at N = 1, the other BASELINE.json configs:
      C2  proteins-shaped GCN aggregation, copy_u-sum F = 32 / 128 / 512;
      C4  rand-100K MLP aggregation, mlp-max d2 = 128 + args (and its ablations);
      C6  the DRAM-bound control: reddit-shaped with uniform sources, F = 512."""
    import torch
    st = S.stream
    fgp = S.fgp
    k_steps = max(3, min(args.steps, 10))

    def timed(fn):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(k_steps + 1)]
        with torch.cuda.stream(st):
            for k in range(k_steps + 1):
                flush.fill_(float(k))
                evs[k][0].record(st)
                fn()
                evs[k][1].record(st)
        sync_all()
        return float(np.mean([evs[k][0].elapsed_time(evs[k][1]) for k in range(1, k_steps + 1)]))

    out = torch.empty_like(S.o256)
    ms = timed(lambda: fgp.gat_attention(S.G, S.X["X256"], S.ydst("X256"), H=H_GAT, out=out, stream=st))
    n, m, F = S.nl, S.m, H_GAT * D_GAT
    b = 8 * (n + 1) + 4 * m + 4 * m * F + 2 * 4 * n * F
    res = {"gat_fused_ms": round(ms, 4), "gat_fused_gbs": round(b / (ms * 1e-3) / 1e9, 1),
           "gat_fused_bytes_model": "8(n+1) + 4m + 4mF + 8nF (X[u] gathered once; Y read, out written)"}
    # bf16 storage (fg_spmm_x16 / fg_sddmm_x16): inputs converted once outside the timing
    X16 = {k: S.X[k].to(torch.bfloat16) for k in ("X512", "X256")}
    lo, nl = S.lo, S.nl
    o512, s1, s8, o256 = (torch.empty_like(S.out512), torch.empty_like(S.s1), torch.empty_like(S.s8),
                          torch.empty_like(S.o256))
    bf = {
        "spmm_copy_u_sum_F512": timed(lambda: fgp.spmm(S.G, "copy_u", "sum", X16["X512"], out=o512, stream=st)),
        "sddmm_u_dot_v_H1_F512": timed(lambda: fgp.sddmm(S.G, X16["X512"], X16["X512"][lo:lo + nl], H=1, out=s1,
                                                         stream=st)),
        "sddmm_u_dot_v_H8_D32": timed(lambda: fgp.sddmm(S.G, X16["X256"], X16["X256"][lo:lo + nl], H=H_GAT,
                                                        out=s8, stream=st)),
        "spmm_u_mul_e_sum_H8_D32": timed(lambda: fgp.spmm(S.G, "u_mul_e", "sum", X16["X256"], H=H_GAT, E=S.s8,
                                                          out=o256, stream=st)),
    }
    res["bf16_storage_ms"] = {k: round(v, 4) for k, v in bf.items()}
    del X16
    # f4: u_dot_v then e_mul (scores scaled by the step's alpha, fused into the write-back)
    s8w = torch.empty_like(S.s8)
    res["sddmm_u_dot_v_e_mul_H8_D32_ms"] = round(timed(
        lambda: fgp.sddmm(S.G, S.X["X256"], S.ydst("X256"), H=H_GAT, E=S.s8, out=s8w, stream=st)), 4)
    res["bf16_storage_note"] = ("row f4: same fp32 arithmetic and outputs, X (and Y) stored as bf16; "
                                "parity vs the oracle on the decoded inputs in tests/test_parity_gpu.py")

    def mlp_impls(G, X8, W, Xd, o, au, ae):
        r = {}
        for name, impl in (("tcgen05_3xtf32", 0), ("tcgen05_bf16_2split", 2), ("ffma_simt", 1)):
            G.tune("mlp_impl", impl)
            r[name] = round(timed(lambda: fgp.spmm(G, "mlp", "max", X8, W=W, X_dst=Xd, out=o, arg_u=au, arg_e=ae,
                                                   stream=st)), 4)
        G.tune("mlp_impl", 0)
        return r

    res["mlp_ablation_reddit_ms"] = mlp_impls(S.G, S.X["X8"], S.W, S.ydst("X8"), S.omlp, S.aumlp, S.aemlp)
    sync_all()
    if world != 1:
        return res
    res["backward"] = run_backward(S, timed, sync_all)
    import gen
    dev = torch.device("cuda")

    def graph_on_gpu(name, uniform=False):
        gg = gen.make_graph(name, uniform_sources=uniform)
        G = fgp.Graph(torch.from_numpy(gg.row_ptr).to(dev), torch.from_numpy(gg.col_idx).to(dev), n_src=gg.n_src)
        return gg, G

    # C2: proteins-shaped GCN aggregation
    gp, Gp = graph_on_gpu("proteins")
    c2 = {}
    for Fp in (32, 128, 512):
        Xp = torch.from_numpy(gen.features((gp.n_src, Fp), gen.feature_seed("proteins"), 0)).to(dev)
        op = torch.empty(gp.n_dst, Fp, device=dev)
        t = timed(lambda: fgp.spmm(Gp, "copy_u", "sum", Xp, out=op, stream=st))
        bts = 8 * (gp.n_dst + 1) + 4 * gp.nnz + 4 * gp.nnz * Fp + 4 * gp.n_dst * Fp
        c2[f"copy_u_sum_F{Fp}"] = {"ms": round(t, 4), "gbs": round(bts / (t * 1e-3) / 1e9, 1)}
        del Xp, op
    res["C2_proteins_gcn"] = c2
    del Gp, gp
    # C4: rand-100K MLP aggregation, d1 = 8, d2 = 128, with args
    gr, Gr = graph_on_gpu("rand100k")
    s4 = gen.feature_seed("rand100k")
    X8 = torch.from_numpy(gen.features((gr.n_src, D1), s4, 3)).to(dev)
    W = torch.from_numpy(gen.features((D1, D2), s4, 4, gen.SCALED, scale=1 / np.sqrt(D1))).to(dev)
    o = torch.empty(gr.n_dst, D2, device=dev)
    au, ae = (torch.empty(gr.n_dst, D2, dtype=torch.int32, device=dev) for _ in range(2))
    abl = mlp_impls(Gr, X8, W, X8, o, au, ae)
    t = abl["tcgen05_3xtf32"]
    res["C4_rand100k_mlp"] = {"ms": t, "tflops": round(mlp_flops(gr.nnz) / (t * 1e-3) / 1e12, 2),
                              "tmem": mlp_roofline(gr.nnz, t, sm_max_mhz()), "ablation_ms": abl}
    X128 = torch.from_numpy(gen.features((gr.n_src, 128), s4, 2)).to(dev)
    o128 = torch.empty(gr.n_dst, 128, device=dev)
    res["C4_rand100k_copy_u_sum_F128_ms"] = round(timed(
        lambda: fgp.spmm(Gr, "copy_u", "sum", X128, out=o128, stream=st)), 4)
    del Gr, gr, X8, W, o, au, ae, X128, o128
    # C6: the control with uniform sources, F = 512: with the L2
    # techniques on (column tiles / source segments, the default) and off ("direct":
    # every gather that misses L2 goes to HBM -- the physical DRAM-bound case)
    gu, Gu = graph_on_gpu("reddit", uniform=True)
    Gu.prepare(F_DOT * 4)
    Xu = S.X["X512"]
    ou = torch.empty(gu.n_dst, F_GCN, device=dev)
    su = torch.empty(gu.nnz, 1, device=dev)
    ob = op_bytes(gu.n_dst, gu.nnz)
    hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)) if \
        os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    ctl = {}
    for variant, knobs in (("uniform", {}), ("uniform_direct", {"l2_tile_mb": 0, "sddmm_seg_mb": 0})):
        for k, v in knobs.items():
            Gu.tune(k, v)
        for name, fn in (("spmm_copy_u_sum_F512", lambda: fgp.spmm(Gu, "copy_u", "sum", Xu, out=ou, stream=st)),
                         ("sddmm_u_dot_v_H1_F512", lambda: fgp.sddmm(Gu, Xu, Xu, H=1, out=su, stream=st))):
            t = timed(fn)
            rec, fresh, _ = ncu_record(name, variant)
            d = {"ms": round(t, 4), "gather_model_gbs": round(ob[name] / (t * 1e-3) / 1e9, 1), "ncu_fresh": bool(fresh)}
            if rec and fresh and rec.get("dram_bytes_per_launch"):
                d["dram_gbs"] = round(rec["dram_bytes_per_launch"] / (t * 1e-3) / 1e9, 1)
                d["dram_frac"] = round(d["dram_gbs"] / hbm, 4)
            ctl[f"{name}_{variant}"] = d
    res["C6_uniform_sources_control"] = ctl
    del Gu, gu, ou, su
    torch.cuda.empty_cache()
    return res


def gpu_local_cpus(torch) -> set | None:
    """The host CPUs on the GPU's NUMA node (sysfs local_cpulist of its PCI
    device), or None."""
    try:
        pr = torch.cuda.get_device_properties(torch.cuda.current_device())
        bus = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        txt = open(f"/sys/bus/pci/devices/{bus}/local_cpulist").read().strip()
        cpus = set()
        for part in txt.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        return cpus & os.sched_getaffinity(0) or None
    except Exception:
        return None


def run_e2e(S, host, args, world, sync_all, flush):
    """Same step through the public API from pinned HOST buffers: H2D of the
    step's inputs, the step, D2H of every op's result, all inside the events
    (copies overlapped with the compute on two copy streams, Step.enqueue_pipelined)."""
    import torch
    st = S.stream
    lo, nl = S.lo, S.nl
    # host side on the GPU's NUMA node: the pinned buffers are allocated (first
    # touch) and the copies issued from there (measured run-to-run e2e spread
    # 58-72 ms without it); the previous affinity is restored at the end
    old_aff = os.sched_getaffinity(0)
    local = gpu_local_cpus(torch)
    if local:
        os.sched_setaffinity(0, local)
    ins = {k: torch.from_numpy(np.ascontiguousarray(host[k][lo:lo + nl])).pin_memory() for k in
           ("X512", "X256", "X128", "X8")}
    w_h = torch.from_numpy(host["W"]).pin_memory()
    outs_d = S.outputs()
    outs_h = {id(o): torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in outs_d}
    h2d = sum(t.numel() * t.element_size() for t in ins.values()) + w_h.numel() * 4
    d2h = sum(t.numel() * t.element_size() for t in outs_h.values())
    k_steps = max(1, args.steps)   # the same K as the device-timed step
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k_steps + 1)]
    s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(st):
        for k in range(k_steps + 1):
            flush.fill_(float(k))
            evs[k][0].record(st)
            s_h2d.wait_event(evs[k][0])
            s_d2h.wait_event(evs[k][0])
            S.enqueue_pipelined(ins, w_h, outs_h, s_h2d, s_d2h)
            st.wait_stream(s_d2h)          # every result is on the host
            evs[k][1].record(st)
    sync_all()
    ms = float(np.mean([evs[k][0].elapsed_time(evs[k][1]) for k in range(1, k_steps + 1)]))
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_bytes = S.total_bytes
    os.sched_setaffinity(0, old_aff)
    return {"value": total_bytes / (ms * 1e-3) / 1e9, "unit": "GB/s",
            "ms_per_step": ms, "h2d_bytes_per_step": int(h2d) * world, "d2h_bytes_per_step": int(d2h) * world,
            "steps": k_steps}


def run_reference(args, world, rank):
    """--impl reference: the fp64 CPU oracle (this tier's reference arm), on
    bounded row samples of the same workload, on the host cores."""
    if world > 1 and rank != 0:
        return
    import gen
    g = gen.make_graph(GRAPH, uniform_sources=args.uniform_sources)
    host = make_inputs(g)
    rows = calibrate_sample(g, host, target_s=4.0)[0]
    for _ in range(args.warmup):
        oracle_sample_step(g, host, rows)
    dts, b, me = [], 0, 0
    for _ in range(args.steps):
        dt, b, me = oracle_sample_step(g, host, rows)
        dts.append(dt)
    dt = float(np.mean(dts))
    value = b / dt / 1e9
    sample = (f"each step: all 7 ops on {rows.size} seeded-random destination rows ({me} in-edges, "
              f"{me / g.nnz:.2%} of the graph); fp64 C oracle, OpenMP over rows")
    line = {
        "metric": metric_name(), "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": "reddit-shaped synthetic graph, same 7-op step as the GPU arm, bounded row sample",
                   "graph": GRAPH, "n": g.n_dst, "nnz": g.nnz, "sample_rows": int(rows.size),
                   "sample_edges": int(me)},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cpu_threads(), "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    sys.exit(main() or 0)
