"""gSpMM launch-knob A/B (dev tool): cases `graph:msg:reduce:F[:args]` with one
fg_graph_tune knob varied on one handle per graph; every variant checked bit
for bit against the first (sum orders never change with these knobs).  CUDA
events, L2 flushed before each launch, median of 7, variants interleaved.

    python tools/spmm_ab.py KNOB v1,v2 reddit:copy_u:sum:512,reddit:copy_u:max:128:args,...
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
cases = [c.split(":") for c in sys.argv[3].split(",")]
graphs = {}


def once(fn):
    flush.fill_(1.0)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e)


for c in cases:
    gname, msg, red, F = c[0], c[1], c[2], int(c[3])
    args = len(c) > 4 and c[4] == "args"
    if gname not in graphs:
        g = gen.make_graph(gname)
        graphs[gname] = (g, fgp.Graph(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda()))
    g, G = graphs[gname]
    H = 8 if msg == "u_mul_e" else 1
    X = torch.from_numpy(gen.features((g.n_src, F), 31, 0)).cuda()
    E = torch.from_numpy(gen.features((g.nnz, H), 31, 1, gen.UNIT)).cuda() if msg == "u_mul_e" else None
    outs = {v: torch.empty(g.n_dst, F, device="cuda") for v in vals}
    au = {v: torch.empty(g.n_dst, F, dtype=torch.int32, device="cuda") if args else None for v in vals}
    ts = {v: [] for v in vals}
    for r in range(8):
        for v in vals:
            G.tune(knob, v)
            kw = dict(arg_u=au[v]) if args else {}
            ms = once(lambda: fgp.spmm(G, msg, red, X, H=H, E=E, out=outs[v], **kw))
            if r:
                ts[v].append(ms)
    G.tune(knob, vals[0])
    for v in vals:
        same = bool(torch.equal(outs[v], outs[vals[0]])) and (not args or bool(torch.equal(au[v], au[vals[0]])))
        print(f"{gname} {msg}-{red} F={F}{' +args' if args else ''} {knob}={v}: {np.median(ts[v]):.3f} ms "
              f"(min {min(ts[v]):.3f})  bitequal={same}", flush=True)
