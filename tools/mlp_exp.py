"""MLP pipeline experiments on the reddit graph (dev tool)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen, paper_2008_11359_b200 as fgp
g = gen.make_graph(sys.argv[1] if len(sys.argv) > 1 else "reddit")
G = fgp.Graph(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
n = g.n_dst
X8 = torch.rand(n, 8, device="cuda"); W = torch.rand(8, 128, device="cuda") - 0.5
o = torch.empty(n, 128, device="cuda"); au = torch.empty(n, 128, dtype=torch.int32, device="cuda"); ae = torch.empty_like(au)
def t(fn, reps=5):
    ts = []
    for i in range(reps + 1):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        if i: ts.append(s.elapsed_time(e))
    return np.median(ts)
for dbg in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "1", "2", "3"]):
    if dbg.startswith("eb"):   # eb<ns>: epilogue wait back-off
        os.environ["FG_MLP_DBG"] = "0"
        os.environ["FG_MLP_EPI_BACKOFF_NS"] = dbg[2:]
    elif dbg.startswith("bo"):   # bo<ns>: back-off sweep with every stage on
        os.environ["FG_MLP_DBG"] = "0"
        os.environ["FG_MLP_BACKOFF_NS"] = dbg[2:]
    else:
        os.environ["FG_MLP_DBG"] = dbg
    print(f"{sys.argv[1] if len(sys.argv)>1 else 'reddit'} dbg={dbg} max+args {t(lambda: fgp.spmm(G, 'mlp', 'max', X8, W=W, out=o, arg_u=au, arg_e=ae)):.3f} ms"
          f"  sum {t(lambda: fgp.spmm(G, 'mlp', 'sum', X8, W=W, out=o)):.3f} ms")
