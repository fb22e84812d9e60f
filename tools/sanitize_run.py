"""Run every libfg entry point once on small graphs (for compute-sanitizer)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen
import paper_2008_11359_b200 as fgp

dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
for g in (gen.make_graph("tiny"), gen.random_graph(600, 30000, 3, sigma=1.5, n_empty=10)):
    G = fgp.Graph(dev(g.row_ptr), dev(g.col_idx))
    GT = G.transpose()
    for F in (4, 16, 128, 512):
        X = dev(gen.features((g.n_src, F), 1, 0))
        fgp.spmm(G, "copy_u", "sum", X)
        fgp.spmm(G, "copy_u", "max", X, arg_u=True, arg_e=True)
        fgp.sddmm(G, X)
    H, D = 8, 32
    X = dev(gen.features((g.n_src, H * D), 2, 0))
    s = fgp.sddmm(G, X, H=H)
    a = fgp.edge_softmax(G, s, H=H)
    fgp.spmm(G, "u_mul_e", "sum", X, H=H, E=a)
    out, au, _ = fgp.spmm(G, "u_mul_e", "max", X, H=H, E=a, arg_u=True, arg_e=True)
    fgp.gat_attention(G, X, H=H)
    fgp.spmm_backward(G, GT, "u_mul_e", "max", out, H=H, X=X, E=a, arg_u=au, want_dE=True)
    fgp.sddmm_backward(G, GT, X, X, s, H=H)
    fgp.edge_softmax_backward(G, a, s, H=H)
    X8 = dev(gen.features((g.n_src, 8), 3, 0))
    W = dev(gen.features((8, 128), 3, 1))
    fgp.spmm(G, "mlp", "max", X8, W=W, arg_u=True, arg_e=True)
    fgp.spmm(G, "mlp", "sum", X8, W=W)
    fgp.spmm(G, "mlp", "max", X8, W=W[:, :32].contiguous(), arg_u=True)   # d2 < 128: idle epilogue warps
    # bf16 feature storage (16-byte pairs and 8-byte chunks) and u_dot_v-then-e_mul
    for F in (8, 32, 128, 512):
        Xb = dev(gen.features((g.n_src, F), 4, 0)).to(torch.bfloat16)
        fgp.spmm(G, "copy_u", "sum", Xb)
        fgp.spmm(G, "copy_u", "max", Xb, arg_u=True, arg_e=True)
        fgp.sddmm(G, Xb)
    Xb = X.to(torch.bfloat16)
    fgp.sddmm(G, Xb, H=H)
    fgp.spmm(G, "u_mul_e", "sum", Xb, H=H, E=a)
    fgp.sddmm(G, X, H=H, E=a)
    X64 = dev(gen.features((g.n_src, 256), 5, 0))
    fgp.sddmm(G, X64, H=64, E=dev(gen.features((g.nnz, 64), 5, 1)))   # H > G: the second-pass scale
torch.cuda.synchronize()
print("sanitize_run: OK")
