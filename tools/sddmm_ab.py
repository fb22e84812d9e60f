"""gSDDMM launch-knob A/B on the reddit-shaped graph (dev tool): u_dot_v at
the given (H, F) shapes with one fg_graph_tune knob varied on ONE prepared
handle; checks every variant against the first bit for bit.  CUDA events, L2
flushed before each launch, median of 7, rounds interleaved.

    python tools/sddmm_ab.py KNOB v1,v2,... [H:F,H:F,...] [graph]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2008_11359_b200 as fgp  # noqa: E402

flush = torch.empty(256 << 20 >> 2, device="cuda")
knob = sys.argv[1]
vals = [int(x) for x in sys.argv[2].split(",")]
shapes = [tuple(int(y) for y in x.split(":")) for x in (sys.argv[3] if len(sys.argv) > 3 else "1:512,1:256,8:256").split(",")]
gname = sys.argv[4] if len(sys.argv) > 4 else "reddit"
g = gen.make_graph(gname)
G = fgp.Graph(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())


def once(fn):
    flush.fill_(1.0)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e)


for H, F in shapes:
    G.prepare(F * 4)
    X = torch.from_numpy(gen.features((g.n_src, F), 21, 0)).cuda()
    outs = {v: torch.empty(g.nnz, H, device="cuda") for v in vals}
    ts = {v: [] for v in vals}
    for r in range(8):
        for v in vals:
            G.tune(knob, v)
            ms = once(lambda: fgp.sddmm(G, X, H=H, out=outs[v]))
            if r:
                ts[v].append(ms)
    G.tune(knob, vals[0])
    for v in vals:
        same = bool(torch.equal(outs[v], outs[vals[0]]))
        print(f"{gname} u_dot_v H={H} F={F} {knob}={v}: {np.median(ts[v]):.3f} ms (min {min(ts[v]):.3f})  bitequal={same}",
              flush=True)
