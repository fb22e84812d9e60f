"""CTA-per-row threshold sweep (dev tool): FG_SPMM_HEAVY_DEG values on reddit copy_u-max
F=128 + args (G=8 column tiles) and rand-100K copy_u-sum F=32 (G=8)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen, paper_2008_11359_b200 as fgp
flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
def t(fn, reps=8):
    ts = []
    for i in range(reps + 1):
        flush.fill_(float(i))
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        if i: ts.append(s.elapsed_time(e))
    return float(np.mean(ts))
cases = []
for gname, F, red in (("reddit", 128, "max"), ("rand100k", 32, "sum"), ("proteins", 32, "sum")):
    g = gen.make_graph(gname)
    G = fgp.Graph(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
    X = torch.rand(g.n_dst, F, device="cuda")
    cases.append((gname, F, red, G, X))
for v in sys.argv[1].split(","):
    if v == "auto":
        os.environ.pop("FG_SPMM_HEAVY_DEG", None)
    else:
        os.environ["FG_SPMM_HEAVY_DEG"] = v
    r = []
    for gname, F, red, G, X in cases:
        if red == "max":
            ms = t(lambda: fgp.spmm(G, "copy_u", "max", X, arg_u=True, arg_e=True))
        else:
            ms = t(lambda: fgp.spmm(G, "copy_u", "sum", X))
        r.append(f"{gname} F{F} {red} {ms:.3f}")
    print(v, " | ".join(r), flush=True)
