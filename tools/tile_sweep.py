"""Sweep FG_L2_TILE_MB for the column-tiled SpMM ops and FG_UMULE_TILE (dev tool)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2008_11359_b200 as fgp  # noqa: E402

g = gen.make_graph("reddit")
G = fgp.Graph(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
n, m = g.n_dst, g.nnz
flush = torch.empty(int(256e6) // 4, dtype=torch.float32, device="cuda")


def timeit(fn, reps=5):
    ts = []
    for i in range(reps + 1):
        flush.fill_(i)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        if i:
            ts.append(s.elapsed_time(e))
    return float(np.median(ts))


X512 = torch.rand(n, 512, device="cuda"); o512 = torch.empty(n, 512, device="cuda")
X128 = torch.rand(n, 128, device="cuda"); o128 = torch.empty(n, 128, device="cuda")
au = torch.empty(n, 128, dtype=torch.int32, device="cuda"); ae = torch.empty_like(au)
X256 = torch.rand(n, 256, device="cuda"); o256 = torch.empty(n, 256, device="cuda")
E = torch.rand(m, 8, device="cuda")
for mb in (0, 24, 32, 48, 64, 96, 128):
    os.environ["FG_L2_TILE_MB"] = str(mb)
    r = [timeit(lambda: fgp.spmm(G, "copy_u", "sum", X512, out=o512)),
         timeit(lambda: fgp.spmm(G, "copy_u", "sum", X128, out=o128)),
         timeit(lambda: fgp.spmm(G, "copy_u", "max", X128, out=o128, arg_u=au, arg_e=ae))]
    os.environ["FG_UMULE_TILE"] = "0"
    r.append(timeit(lambda: fgp.spmm(G, "u_mul_e", "sum", X256, H=8, E=E, out=o256)))
    os.environ["FG_UMULE_TILE"] = "1"
    r.append(timeit(lambda: fgp.spmm(G, "u_mul_e", "sum", X256, H=8, E=E, out=o256)))
    os.environ["FG_UMULE_TILE"] = "0"
    print(f"tile_mb={mb:4d}  sum F512 {r[0]:7.3f}  sum F128 {r[1]:7.3f}  max F128 {r[2]:7.3f}  "
          f"u_mul_e H8 {r[3]:7.3f}  u_mul_e H8 tiled {r[4]:7.3f} ms", flush=True)
