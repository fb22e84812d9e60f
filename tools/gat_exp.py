"""Fused-GAT launch variants on the reddit graph (dev tool): FG_GAT_VARIANT sweep."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen, paper_2008_11359_b200 as fgp
g = gen.make_graph(sys.argv[1] if len(sys.argv) > 1 else "reddit")
G = fgp.Graph(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
n, H, D = g.n_dst, 8, 32
X = torch.rand(n, H * D, device="cuda") - 0.5
out = torch.empty_like(X)
flush = torch.empty(int(256e6) // 4, device="cuda")
def t(fn, reps=5):
    ts = []
    for i in range(reps + 1):
        flush.fill_(i)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        if i: ts.append(s.elapsed_time(e))
    return np.median(ts)
ref = None
for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0"]):
    os.environ["FG_GAT_HEAVY_DEG"] = v
    ms = t(lambda: fgp.gat_attention(G, X, X, H=H, out=out))
    o = out.clone()
    if ref is None: ref = o
    print(f"variant {v}: {ms:.3f} ms  max|diff vs first| {float((o - ref).abs().max()):.3e}", flush=True)
