"""Table tab:gpu-kernel on B200: GCN aggregation (copy_u-sum gSpMM), MLP
aggregation (mlp-max gSpMM, d1 = 8, d2 = F) and dot-product attention (u_dot_v
gSDDMM) on the proteins-, reddit- and rand-100K-shaped synthetic graphs at
F = 32 .. 512, fp32 (and bf16 feature storage for GCN / attention).

    python tools/sweep.py [out_prefix]      -> <out_prefix>.json and .md

Protocol as the paper's: one warm-up, mean of 10 runs, CUDA events; L2
flushed (256 MB write) before every run.  The paper's V100 numbers (BASELINE.md
§2, Table tab:gpu-kernel P:727-814) are printed beside ours as CONTEXT: the
real graphs have community locality the synthetic ones do not.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2008_11359_b200 as fgp  # noqa: E402

FS = [32, 64, 128, 256, 512]
V100 = {  # BASELINE.md §2 (FeatGraph rows of Table tab:gpu-kernel), ms
    ("gcn", "proteins"): [4.6, 7.8, 15.4, 30.8, 61.9], ("gcn", "reddit"): [14.3, 28.6, 57.8, 116.9, 232.0],
    ("gcn", "rand100k"): [2.8, 4.9, 10.2, 20.3, 39.9],
    ("mlp", "proteins"): [26.9, 46.7, 87.4, 168.9, 332.9], ("mlp", "reddit"): [33.2, 76.7, 142.9, 277.1, 547.9],
    ("mlp", "rand100k"): [8.9, 14.9, 26.0, 46.6, 89.6],
    ("attn", "proteins"): [24.4, 37.9, 69.3, 143.3, 333.7], ("attn", "reddit"): [35.9, 56.6, 103.7, 212.0, 483.2],
    ("attn", "rand100k"): [14.9, 23.2, 42.3, 87.8, 201.5],
}


def timed(fn, flush, reps=10):
    ts = []
    for i in range(reps + 1):
        flush.fill_(float(i))
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        if i:
            ts.append(s.elapsed_time(e))
    return float(np.mean(ts))


def main():
    prefix = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep"
    flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
    rows = []
    for gname in ("proteins", "reddit", "rand100k"):
        g = gen.make_graph(gname)
        G = fgp.Graph(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
        n, m = g.n_dst, g.nnz
        s = gen.feature_seed(gname)
        X8 = torch.from_numpy(gen.features((n, 8), s, 3)).cuda()
        for fi, F in enumerate(FS):
            X = torch.from_numpy(gen.features((n, F), s, 10 + fi)).cuda()
            Xb = X.to(torch.bfloat16)
            W = torch.from_numpy(gen.features((8, F), s, 4, gen.SCALED, scale=1 / np.sqrt(8))).cuda()
            out = torch.empty(n, F, device="cuda")
            sc = torch.empty(m, 1, device="cuda")
            idx = 8 * (n + 1) + 4 * m
            b_gcn = idx + 4 * m * F + 4 * n * F
            b_att = idx + 4 * m * F + 4 * n * F + 4 * m
            r = {"graph": gname, "n": n, "nnz": m, "F": F}
            r["gcn_ms"] = timed(lambda: fgp.spmm(G, "copy_u", "sum", X, out=out), flush)
            r["gcn_bf16_ms"] = timed(lambda: fgp.spmm(G, "copy_u", "sum", Xb, out=out), flush)
            r["mlp_ms"] = timed(lambda: fgp.spmm(G, "mlp", "max", X8, W=W, out=out), flush)
            r["attn_ms"] = timed(lambda: fgp.sddmm(G, X, H=1, out=sc), flush)
            r["attn_bf16_ms"] = timed(lambda: fgp.sddmm(G, Xb, H=1, out=sc), flush)
            r["gcn_gbs"] = b_gcn / (r["gcn_ms"] * 1e-3) / 1e9
            r["attn_gbs"] = b_att / (r["attn_ms"] * 1e-3) / 1e9
            r["mlp_tflops"] = 2 * m * 8 * F / (r["mlp_ms"] * 1e-3) / 1e12
            for k in ("gcn", "mlp", "attn"):
                r[f"{k}_v100_ms"] = V100[(k, gname)][fi]
            rows.append(r)
            print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
        del G
    json.dump(rows, open(prefix + ".json", "w"), indent=1)
    lines = ["| kernel | graph | " + " | ".join(f"F={F}" for F in FS) + " |", "|---|---|" + "---|" * len(FS)]
    for k, nm in (("gcn", "GCN copy_u-sum"), ("attn", "attention u_dot_v"), ("mlp", "MLP mlp-max (d1=8)")):
        for gname in ("proteins", "reddit", "rand100k"):
            rs = [r for r in rows if r["graph"] == gname]
            cells = []
            for r in rs:
                c = f"{r[k + '_ms']:.2f}"
                if k in ("gcn", "attn"):
                    c += f" / {r[k + '_bf16_ms']:.2f}"
                c += f" ({r[k + '_v100_ms']:.1f})"
                cells.append(c)
            lines.append(f"| {nm} | {gname} | " + " | ".join(cells) + " |")
    open(prefix + ".md", "w").write(
        "B200 ms per op, fp32 / bf16-storage (paper V100 ms in parentheses, context only)\n\n" + "\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
