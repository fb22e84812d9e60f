"""Launch-variant sweep on the reddit graph (dev tool):
    python tools/var_exp.py ENVVAR v1,v2,...   (times sddmm H1 F512, sddmm H8 D32, u_mul_e H8 D32, copy_u-sum F512)"""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen, paper_2008_11359_b200 as fgp
g = gen.make_graph("reddit")
G = fgp.Graph(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
n, m = g.n_dst, g.nnz
X512 = torch.rand(n, 512, device="cuda") - 0.5
X256 = torch.rand(n, 256, device="cuda") - 0.5
E8 = torch.rand(m, 8, device="cuda")
s1, s8 = torch.empty(m, 1, device="cuda"), torch.empty(m, 8, device="cuda")
o512, o256 = torch.empty(n, 512, device="cuda"), torch.empty(n, 256, device="cuda")
flush = torch.empty(int(256e6) // 4, device="cuda")
def t(fn, reps=5):
    ts = []
    for i in range(reps + 1):
        flush.fill_(i)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        if i: ts.append(s.elapsed_time(e))
    return np.median(ts)
var = sys.argv[1]
for v in sys.argv[2].split(","):
    os.environ[var] = v
    r = [t(lambda: fgp.sddmm(G, X512, H=1, out=s1)), t(lambda: fgp.sddmm(G, X256, H=8, out=s8)),
         t(lambda: fgp.spmm(G, "u_mul_e", "sum", X256, H=8, E=E8, out=o256)),
         t(lambda: fgp.spmm(G, "copy_u", "sum", X512, out=o512))]
    print(f"{var}={v}: sddmm_H1_F512 {r[0]:.3f}  sddmm_H8 {r[1]:.3f}  u_mul_e_H8 {r[2]:.3f}  copy_u_sum_F512 {r[3]:.3f} ms",
          flush=True)
