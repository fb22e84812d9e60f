"""Sweep the L2-tiling knobs (FG_L2_TILE_MB, FG_SDDMM_L2_TILE, FG_SDDMM_SEGMENT) on
the reddit-shaped graph at F=512 (development tool)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2008_11359_b200 as fgp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "reddit"
g = gen.make_graph(name)
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


def setenv(**kw):
    for k in ("FG_L2_TILE_MB", "FG_SDDMM_L2_TILE", "FG_SDDMM_SEGMENT", "FG_SDDMM_PERSIST", "FG_SDDMM_SEG_MB"):
        os.environ.pop(k, None)
    for k, v in kw.items():
        os.environ[k] = str(v)


X = torch.rand(n, 512, device="cuda")
out = torch.empty(n, 512, device="cuda")
s1 = torch.empty(m, 1, device="cuda")
only_sddmm = "--sddmm" in sys.argv
for mb in (() if only_sddmm else (0, 16, 24, 32, 48, 64, 96, 128)):
    setenv(FG_L2_TILE_MB=mb)
    print(f"copy_u_sum F512 tile_mb={mb:4d}  {timeit(lambda: fgp.spmm(G, 'copy_u', 'sum', X, out=out)):7.3f} ms", flush=True)
setenv()
print(f"sddmm H1 F512 untiled          {timeit(lambda: fgp.sddmm(G, X, H=1, out=s1)):7.3f} ms", flush=True)
for mb in (() if only_sddmm else (16, 32, 48, 64, 96, 128)):
    setenv(FG_L2_TILE_MB=mb, FG_SDDMM_L2_TILE=1)
    print(f"sddmm H1 F512 coltile mb={mb:4d}  {timeit(lambda: fgp.sddmm(G, X, H=1, out=s1)):7.3f} ms", flush=True)
X256 = torch.rand(n, 256, device="cuda")
s8 = torch.empty(m, 8, device="cuda")
for mb in (0, 24, 32, 48, 64, 96):
    setenv(FG_SDDMM_SEG_MB=mb)
    t1 = timeit(lambda: fgp.sddmm(G, X, H=1, out=s1))
    t8 = timeit(lambda: fgp.sddmm(G, X256, H=8, out=s8))
    print(f"sddmm segmented persistent seg_mb={mb:4d}  H1 F512 {t1:7.3f} ms   H8 D32 {t8:7.3f} ms", flush=True)
