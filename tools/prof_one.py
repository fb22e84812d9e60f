"""Run one op a few times on the reddit graph (for ncu -k filtering)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen, paper_2008_11359_b200 as fgp
op = sys.argv[1]
g = gen.make_graph("reddit")
G = fgp.Graph(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
n = g.n_dst
if op == "mlp":
    X8 = torch.rand(n, 8, device="cuda"); W = torch.rand(8, 128, device="cuda") - 0.5
    o = torch.empty(n, 128, device="cuda"); au = torch.empty(n, 128, dtype=torch.int32, device="cuda")
    for _ in range(3): fgp.spmm(G, "mlp", "max", X8, W=W, out=o, arg_u=au)
elif op == "sddmm512":
    X = torch.rand(n, 512, device="cuda"); s1 = torch.empty(g.nnz, 1, device="cuda")
    for _ in range(2): fgp.sddmm(G, X, H=1, out=s1)
elif op == "gat":
    X = torch.rand(n, 256, device="cuda") * 0.25; o = torch.empty(n, 256, device="cuda")
    for _ in range(3): fgp.gat_attention(G, X, H=8, out=o)
torch.cuda.synchronize()
