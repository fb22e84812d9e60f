"""The paper's ablations on B200, one gpurun call:

  E7  hybrid partitioning (measured by the paper on
      rand-100K GCN, 10-20 %): copy_u-sum F = 32 / 128 on the
      rand-100K-, reddit- and proteins-shaped graphs, plain vs the hottest
      sources staged in shared memory (8 / 24 / 48 / 96 KB per CTA);
  E6  gSDDMM dot products: lanes over features + shuffle reduction (ours) vs
      thread-per-edge, F = 32 .. 512 on reddit.

    python tools/ablations.py out_prefix   -> out_prefix.json / .md
Protocol: CUDA events, L2 flushed (256 MB write) before each run, 1 warm-up +
median of 7; the plain and ablated launches alternate on the same handle."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2008_11359_b200 as fgp  # noqa: E402

flush = torch.empty(64 << 20, device="cuda")


def t(fn, reps=7):
    ts = []
    for i in range(reps + 1):
        flush.fill_(i)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        if i:
            ts.append(s.elapsed_time(e))
    return float(np.median(ts))


out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", "ablations") \
    if len(sys.argv) < 2 else sys.argv[1]
res = {"E7_hybrid": {}, "E6_sddmm_dot": {}}
md = ["# Ablations on one B200 (tools/ablations.py)", ""]
md += ["## E7 hybrid partitioning (copy_u-sum; ms, plain vs staged hot sources)", "",
       "| graph | F | plain | 8 KB | 24 KB | 48 KB | 96 KB | hot-edge share at 48 KB |", "|---|---|---|---|---|---|---|---|"]
for name in ("rand100k", "reddit", "proteins"):
    g = gen.make_graph(name)
    G = fgp.Graph(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
    for F in (32, 128):
        X = torch.from_numpy(gen.features((g.n_src, F), 9, 0)).cuda()
        o = torch.empty(g.n_dst, F, device="cuda")
        row = {"plain": t(lambda: fgp.spmm(G, "copy_u", "sum", X, out=o))}
        ref = o.clone()
        share48 = None
        for kb in (8, 24, 48, 96):
            G.prepare_hybrid(F * 4, kb * 1024)
            G.tune("hybrid", 1)
            row[f"{kb}KB"] = t(lambda: fgp.spmm(G, "copy_u", "sum", X, out=o))
            assert torch.equal(o, ref), "hybrid result differs"
            k, share = G.hybrid_info()
            row[f"{kb}KB_hot_rows"], row[f"{kb}KB_hot_share"] = k, share
            if kb == 48:
                share48 = share
            G.tune("hybrid", 0)
        res["E7_hybrid"][f"{name}_F{F}"] = row
        md.append(f"| {name} | {F} | {row['plain']:.3f} | {row['8KB']:.3f} | {row['24KB']:.3f} | {row['48KB']:.3f} | "
                  f"{row['96KB']:.3f} | {share48:.3f} |")
        print(name, F, row, flush=True)
    del G
md += ["", "## E6 gSDDMM dot product (u_dot_v, reddit; ms)", "",
       "| H x D | shuffle reduction (ours) | thread per edge | ratio |", "|---|---|---|---|"]
g = gen.make_graph("reddit")
G = fgp.Graph(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
for H, D in ((1, 32), (1, 128), (1, 512), (8, 32)):
    G.prepare(H * D * 4)
    X = torch.from_numpy(gen.features((g.n_src, H * D), 11, 0)).cuda()
    s = torch.empty(g.nnz, H, device="cuda")
    a = t(lambda: fgp.sddmm(G, X, H=H, out=s))
    G.tune("sddmm_dot", 1)
    b = t(lambda: fgp.sddmm(G, X, H=H, out=s))
    G.tune("sddmm_dot", 0)
    res["E6_sddmm_dot"][f"H{H}_D{D}"] = {"shuffle_ms": a, "thread_per_edge_ms": b}
    md.append(f"| {H} x {D} | {a:.3f} | {b:.3f} | {b / a:.2f}x |")
    print("E6", H, D, a, b, flush=True)
json.dump(res, open(out + ".json", "w"), indent=1)
open(out + ".md", "w").write("\n".join(md) + "\n")
