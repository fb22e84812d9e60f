"""u_dot_v H=1 segment-budget sweep at F = 64..512 (dev tool): FG_SDDMM_SEG_MB values."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen, paper_2008_11359_b200 as fgp
flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
def t(fn, reps=5):
    ts = []
    for i in range(reps + 1):
        flush.fill_(float(i))
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        if i: ts.append(s.elapsed_time(e))
    return float(np.mean(ts))
for gname in sys.argv[1].split(","):
    g = gen.make_graph(gname)
    G = fgp.Graph(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
    sc = torch.empty(g.nnz, 1, device="cuda")
    for F in (64, 128, 256, 512):
        X = torch.rand(g.n_dst, F, device="cuda") - 0.5
        Xb = X.to(torch.bfloat16)
        res = []
        for mb in sys.argv[2].split(","):
            os.environ["FG_SDDMM_SEG_MB"] = mb
            res.append(f"seg{mb}: {t(lambda: fgp.sddmm(G, X, H=1, out=sc)):.2f}/{t(lambda: fgp.sddmm(G, Xb, H=1, out=sc)):.2f}")
        print(gname, F, "  ".join(res), flush=True)
    X8 = torch.rand(g.n_dst, 8, device="cuda") - 0.5
    for d2 in (32, 64, 128):
        W = torch.rand(8, d2, device="cuda") - 0.5
        o = torch.empty(g.n_dst, d2, device="cuda")
        print(gname, "mlp d2", d2, f"{t(lambda: fgp.spmm(G, 'mlp', 'max', X8, W=W, out=o)):.2f}", flush=True)
