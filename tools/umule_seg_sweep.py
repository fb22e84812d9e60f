"""u_mul_e-sum source-segment sweep (dev tool): reddit-shaped
graph, H=8 D=32, with the segment budget (fg_graph_tune spmm_seg_mb, then
fg_graph_prepare) varied on one handle.  CUDA events, L2 flushed before each
launch, median of 7.  `--once MB` runs a single call (for ncu).

    python tools/umule_seg_sweep.py [mb,mb,...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2008_11359_b200 as fgp  # noqa: E402

flush = torch.empty(256 << 20 >> 2, device="cuda")


def t(fn, reps=7):
    ts = []
    for i in range(reps + 1):
        flush.fill_(float(i))
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        if i:
            ts.append(s.elapsed_time(e))
    return float(np.median(ts))


once = "--once" in sys.argv
args = [a for a in sys.argv[1:] if a != "--once"]
mbs = [int(x) for x in (args[0] if args else "0,24,32,48,64,80").split(",")]
g = gen.make_graph("reddit")
G = fgp.Graph(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
H, D = 8, 32
F = H * D
X = torch.from_numpy(gen.features((g.n_src, F), 7, 0)).cuda()
E = torch.from_numpy(gen.features((g.nnz, H), 7, 1, gen.UNIT)).cuda()
out = torch.empty(g.n_dst, F, device="cuda")
ref = None
for mb in mbs:
    G.tune("spmm_seg_mb", mb)
    G.prepare(F * 4)
    if once:
        flush.fill_(1.0)
        fgp.spmm(G, "u_mul_e", "sum", X, H=H, E=E, out=out)
        torch.cuda.synchronize()
        continue
    ms = t(lambda: fgp.spmm(G, "u_mul_e", "sum", X, H=H, E=E, out=out))
    if ref is None:
        ref = out.clone()
    err = float((out - ref).abs().max())
    print(f"reddit u_mul_e-sum H={H} D={D} spmm_seg_mb={mb}: {ms:.3f} ms  max|diff vs first| {err:.3g}", flush=True)
