"""fp32 vs bf16-storage timing on the reddit graph (dev tool):
    python tools/bf16_exp.py [ENVVAR v1,v2,...]"""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen, paper_2008_11359_b200 as fgp
g = gen.make_graph("reddit")
G = fgp.Graph(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
n, m = g.n_dst, g.nnz
X = {512: torch.rand(n, 512, device="cuda") - 0.5, 256: torch.rand(n, 256, device="cuda") - 0.5,
     128: torch.rand(n, 128, device="cuda") - 0.5}
Xb = {k: v.to(torch.bfloat16) for k, v in X.items()}
s1 = torch.empty(m, 1, device="cuda")
o = {k: torch.empty(n, k, device="cuda") for k in X}
flush = torch.empty(int(256e6) // 4, device="cuda")
def t(fn, reps=5):
    ts = []
    for i in range(reps + 1):
        flush.fill_(i)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        if i: ts.append(s.elapsed_time(e))
    return np.median(ts)
var, vals = (sys.argv[1], sys.argv[2].split(",")) if len(sys.argv) > 2 else (None, [None])
for v in vals:
    if var: os.environ[var] = v
    r = []
    for F in (512, 256, 128):
        r.append(f"copy_u F{F} f32 {t(lambda: fgp.spmm(G, 'copy_u', 'sum', X[F], out=o[F])):.2f} "
                 f"bf16 {t(lambda: fgp.spmm(G, 'copy_u', 'sum', Xb[F], out=o[F])):.2f}")
    for F in (512, 128):
        r.append(f"u_dot_v F{F} f32 {t(lambda: fgp.sddmm(G, X[F], H=1, out=s1)):.2f} "
                 f"bf16 {t(lambda: fgp.sddmm(G, Xb[F], H=1, out=s1)):.2f}")
    print(f"{var}={v}: " + " | ".join(r), flush=True)
