"""Quick per-op timing on a named graph (development tool; bench.py is the contract)."""
import sys, time, json
import numpy as np
import torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import gen
import paper_2008_11359_b200 as fgp

name = sys.argv[1] if len(sys.argv) > 1 else "reddit"
uniform = "--uniform" in sys.argv
t = time.time()
g = gen.make_graph(name, uniform_sources=uniform)
print(f"gen {name} n={g.n_dst} m={g.nnz} {time.time()-t:.1f}s", flush=True)
rp = torch.from_numpy(g.row_ptr).cuda(); ci = torch.from_numpy(g.col_idx).cuda()
t = time.time(); G = fgp.Graph(rp, ci, validate=True); torch.cuda.synchronize(); print(f"graph_create {time.time()-t:.2f}s")
n, m = g.n_dst, g.nnz
flush = torch.empty(int(256e6) // 4, dtype=torch.float32, device="cuda")

def timeit(fn, reps=5):
    ts = []
    for i in range(reps + 1):
        flush.fill_(i)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        if i: ts.append(s.elapsed_time(e))
    return float(np.median(ts))

res = {}
for F in (32, 128, 512):
    X = torch.rand(n, F, device="cuda"); out = torch.empty(n, F, device="cuda")
    ms = timeit(lambda: fgp.spmm(G, "copy_u", "sum", X, out=out))
    B = 4*(n+1) + 4*m + m*F*4 + n*F*4
    res[f"copy_u_sum_F{F}"] = (ms, B/ms/1e6)
for F in (128, 512):
    X = torch.rand(n, F, device="cuda"); out = torch.empty(m, 1, device="cuda")
    ms = timeit(lambda: fgp.sddmm(G, X, H=1, out=out))
    B = 4*(n+1) + 4*m + m*F*4 + n*F*4 + m*4
    res[f"sddmm_H1_F{F}"] = (ms, B/ms/1e6)
X = torch.rand(n, 128, device="cuda"); out = torch.empty(n, 128, device="cuda")
au = torch.empty(n, 128, dtype=torch.int32, device="cuda"); ae = torch.empty_like(au)
ms = timeit(lambda: fgp.spmm(G, "copy_u", "max", X, out=out, arg_u=au, arg_e=ae))
res["copy_u_max_F128_args"] = (ms, (4*(n+1)+4*m+m*512+3*n*512)/ms/1e6)
H, D = 8, 32
X = torch.rand(n, H*D, device="cuda"); s = torch.empty(m, H, device="cuda"); o = torch.empty(n, H*D, device="cuda")
res["gat_sddmm"] = (timeit(lambda: fgp.sddmm(G, X, H=H, out=s)), None)
res["gat_softmax"] = (timeit(lambda: fgp.edge_softmax(G, s, H=H, out=s)), None)
res["gat_umule"] = (timeit(lambda: fgp.spmm(G, "u_mul_e", "sum", X, H=H, E=s, out=o)), None)
X8 = torch.rand(n, 8, device="cuda"); W = torch.rand(8, 128, device="cuda")
o = torch.empty(n, 128, device="cuda")
res["mlp_max_d128"] = (timeit(lambda: fgp.spmm(G, "mlp", "max", X8, W=W, out=o, arg_u=au, arg_e=ae)), None)
for k, (ms, gbs) in res.items():
    print(f"{k:24s} {ms:8.3f} ms  " + (f"{gbs:8.1f} GB/s" if gbs else ""))
Xg = torch.rand(n, 256, device="cuda") * 0.25
og = torch.empty(n, 256, device="cuda")
ms = timeit(lambda: fgp.gat_attention(G, Xg, H=8, out=og))
print(f"{'gat_fused':24s} {ms:8.3f} ms")
