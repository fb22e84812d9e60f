"""MLP (tcgen05) timing on a named graph for A/B of library variants (dev tool):

    FG_LIBFG=... python tools/mlp_exp.py reddit
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2008_11359_b200 as fgp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "reddit"
g = gen.make_graph(name)
G = fgp.Graph(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
n = g.n_dst
X8 = torch.from_numpy(gen.features((n, 8), 5, 3)).cuda()
W = torch.from_numpy(gen.features((8, 128), 5, 4, gen.SCALED, scale=0.35)).cuda()
o = torch.empty(n, 128, device="cuda")
au = torch.empty(n, 128, dtype=torch.int32, device="cuda")
ae = torch.empty_like(au)
flush = torch.empty(64 << 20, device="cuda")


def t(fn, reps=7):
    ts = []
    for i in range(reps + 1):
        flush.fill_(i)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        if i:
            ts.append(s.elapsed_time(e))
    return float(np.median(ts))


lib = os.path.basename(os.environ.get("FG_LIBFG", "libfg.so"))
for impl in (0, 2):
    G.tune("mlp_impl", impl)
    print(f"{name} {lib} impl={impl} max+args {t(lambda: fgp.spmm(G, 'mlp', 'max', X8, W=W, out=o, arg_u=au, arg_e=ae)):.3f} ms"
          f"  sum {t(lambda: fgp.spmm(G, 'mlp', 'sum', X8, W=W, out=o)):.3f} ms", flush=True)
