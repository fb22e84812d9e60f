"""One u_dot_v F=128 launch in fp32 and one in bf16 storage (for ncu)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen, paper_2008_11359_b200 as fgp
g = gen.make_graph("reddit")
G = fgp.Graph(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
X = torch.rand(g.n_dst, 128, device="cuda") - 0.5
Xb = X.to(torch.bfloat16)
s1 = torch.empty(g.nnz, 1, device="cuda")
for _ in range(2):
    fgp.sddmm(G, X, H=1, out=s1)
    fgp.sddmm(G, Xb, H=1, out=s1)
torch.cuda.synchronize()
