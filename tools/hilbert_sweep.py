"""Segmented gSDDMM traversal order sweep (dev tool; DESIGN.md §6/§9, row f3):
segment-major units vs 2D (destination block x source segment) tiles in
Hilbert-curve order, reddit-shaped u_dot_v.  Each config
is `order:seg_mb:rb_mb`; one handle, tables built by fg_graph_prepare per
config; bit-equality against the first config; CUDA events, L2 flushed, median
of 7, configs interleaved per round.

    python tools/hilbert_sweep.py [cfg,cfg,...] [H:F,...] [graph] [--once]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2008_11359_b200 as fgp  # noqa: E402

once_only = "--once" in sys.argv
argv = [a for a in sys.argv[1:] if a != "--once"]
cfgs = [tuple(int(y) for y in c.split(":")) for c in (argv[0] if argv else "0:48:0,1:48:48,1:32:32,1:24:24,1:48:16,1:32:16").split(",")]
shapes = [tuple(int(y) for y in x.split(":")) for x in (argv[1] if len(argv) > 1 else "1:512,8:256").split(",")]
gname = argv[2] if len(argv) > 2 else "reddit"
g = gen.make_graph(gname)
G = fgp.Graph(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
flush = torch.empty(256 << 20 >> 2, device="cuda")


def setcfg(c):
    G.tune("sddmm_order", c[0])
    G.tune("sddmm_seg_mb", c[1])
    G.tune("sddmm_rb_mb", c[2])


def once(fn):
    flush.fill_(1.0)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e)


for H, F in shapes:
    X = torch.from_numpy(gen.features((g.n_src, F), 21, 0)).cuda()
    for c in cfgs:
        setcfg(c)
        G.prepare(F * 4)
    outs = {c: torch.empty(g.nnz, H, device="cuda") for c in cfgs}
    ts = {c: [] for c in cfgs}
    for r in range(1 if once_only else 8):
        for c in cfgs:
            setcfg(c)
            ms = once(lambda: fgp.sddmm(G, X, H=H, out=outs[c]))
            if r:
                ts[c].append(ms)
    if once_only:
        continue
    for c in cfgs:
        same = bool(torch.equal(outs[c], outs[cfgs[0]]))
        print(f"{gname} u_dot_v H={H} F={F} order={c[0]} seg_mb={c[1]} rb_mb={c[2]}: {np.median(ts[c]):.3f} ms "
              f"(min {min(ts[c]):.3f})  bitequal={same}", flush=True)
