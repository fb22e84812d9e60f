"""gSDDMM source-segment sweep (dev tool; DESIGN.md §6 / §9): u_dot_v on the
reddit-shaped graph at H=1 F=512 and H=8 D=32 with the segment budget
(fg_graph_tune sddmm_seg_mb, then fg_graph_prepare) and the persistent CTAs per
SM (sddmm_persist) varied on ONE handle.  CUDA events, L2 flushed before each
launch, median of 5.

    python tools/seg_sweep.py [graph] [mb,mb,...] [persist,...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2008_11359_b200 as fgp  # noqa: E402

flush = torch.empty(256 << 20 >> 2, device="cuda")


def t(fn, reps=5):
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


gname = sys.argv[1] if len(sys.argv) > 1 else "reddit"
mbs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,8,12,16,24,32,48,64").split(",")]
pers = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "-1").split(",")]
g = gen.make_graph(gname)
G = fgp.Graph(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
torch.manual_seed(0)
for F, H in ((512, 1), (256, 8)):
    X = torch.rand(g.n_dst, F, device="cuda") - 0.5
    sc = torch.empty(g.nnz, H, device="cuda")
    ref = None
    for mb in mbs:
        G.tune("sddmm_seg_mb", mb)
        G.prepare(F * 4)
        for p in pers:
            G.tune("sddmm_persist", p)
            ms = t(lambda: fgp.sddmm(G, X, H=H, out=sc))
            if ref is None:
                ref = sc.clone()
            same = bool(torch.equal(ref, sc))
            print(f"{gname} F={F} H={H} seg_mb={mb} persist={p}: {ms:.3f} ms  bitequal={same}", flush=True)
    G.tune("sddmm_seg_mb", 48)
    G.tune("sddmm_persist", -1)
