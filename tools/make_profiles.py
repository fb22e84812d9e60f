"""Turn the ncu captures of one round into the committed summaries under profiles/.

    python tools/make_profiles.py r01c

Reads gpurun_out/prof_{spmm,sddmm,softmax,mlp,gat}_<tag>.ncu-rep (the default
step) and prof_{uspmm,usddmm}_<tag>.ncu-rep (the uniform-sources control) and
gpurun_out/launches_<tag>.csv; writes
  profiles/ncu_summary_<tag>.md    per-kernel metrics (time, DRAM bytes, L2 hit,
                                   occupancy, issue, tensor pipe, top stalls)
  profiles/ncu_traffic.json        per-launch DRAM / L2 bytes and ncu's L2
                                   throughput share per bench op, stamped with
                                   the source hash of the libfg.so captured
                                   (bench.py refuses a capture of another build)
  profiles/launches_<tag>.md       per-launch device times of one bench step
"""
import csv
import gzip
import json
import os
import shutil
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summarise  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_11359_b200.build import source_hash  # noqa: E402
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
OPS_BY_FILE = {   # file key -> (variant, ops in capture order)
    "spmm": ("default", ["spmm_copy_u_sum_F512", "spmm_u_mul_e_sum_H8_D32", "spmm_copy_u_max_F128_args"]),
    "sddmm": ("default", ["sddmm_u_dot_v_H1_F512", "sddmm_u_dot_v_H8_D32"]),
    "softmax": ("default", ["edge_softmax_H8"]),
    "mlp": ("default", ["spmm_mlp_max_d8_d128_args"]),
    "gat": ("default", ["extra_gat_fused_H8_D32"]),
    "uspmm": ("uniform", ["spmm_copy_u_sum_F512"]),
    "usddmm": ("uniform", ["sddmm_u_dot_v_H1_F512"]),
    "dspmm": ("uniform_direct", ["spmm_copy_u_sum_F512"]),
    "dsddmm": ("uniform_direct", ["sddmm_u_dot_v_H1_F512"]),
}


def num(s):
    try:
        v, u = s.split(" ", 1)
        v = float(v.replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ms": 1e-3, "us": 1e-6,
                 "ns": 1e-9, "s": 1.0}.get(u.strip(), 1.0)
        return v * scale
    except Exception:
        return None


lines = [f"# ncu --set full summaries ({tag})", "",
         "Captured with `ncu --set full --clock-control none --import-source on` on one B200 (gpurun), "
         "kernels of one timed `bench.py` step (reddit-shaped graph, 232,965 v / 114,615,892 e). "
         "Times are ncu replay times (cold-cache, serialised), not bench values.", ""]
traffic = {"build_hash": os.environ.get("FG_BUILD_HASH") or source_hash(), "capture": tag,
           "default": {}, "uniform": {}, "uniform_direct": {}}
found = 0
for key, (variant, ops) in OPS_BY_FILE.items():
    path = os.path.join(ROOT, "gpurun_out", f"prof_{key}_{tag}.ncu-rep")
    if not os.path.exists(path) and os.path.exists(path + ".gz"):
        # captures travel back gzip'd (gpurun_out/ is capped at 64 MiB per call)
        tmp = os.path.join(tempfile.gettempdir(), os.path.basename(path))
        with gzip.open(path + ".gz", "rb") as fi, open(tmp, "wb") as fo:
            shutil.copyfileobj(fi, fo)
        path = tmp
    if not os.path.exists(path):
        continue
    found += 1
    for op, d in zip(ops, summarise(path)):
        t = num(d.get("gpu__time_duration.sum", ""))
        rd = num(d.get("dram__bytes_read.sum", "")) or 0.0
        wr = num(d.get("dram__bytes_write.sum", "")) or 0.0
        lts = num(d.get("lts__t_sectors.sum", "").replace(" sector", " byte"))
        lts = lts * 32 if lts else None
        lpct = d.get("lts__throughput.avg.pct_of_peak_sustained_elapsed", "")
        try:
            lpct = float(lpct.split()[0].replace(",", ""))
        except (ValueError, IndexError):
            lpct = None
        traffic[variant][op] = {"kernel": d["kernel"], "dram_bytes_per_launch": rd + wr, "dram_read": rd,
                                "dram_write": wr, "l2_bytes_per_launch": lts, "lts_throughput_pct": lpct,
                                "ncu_time_s": t, "dram_gbs": (rd + wr) / t / 1e9 if t else None,
                                "l2_hit_pct": d.get("lts__t_sector_hit_rate.pct"), "capture": f"prof_{key}_{tag}"}
        lines += [f"## {op}" + {"default": "", "uniform": " (uniform-sources control)",
                                 "uniform_direct": " (uniform sources, L2 tiling / segments off)"}[variant], "",
                  f"`{d['kernel']}`", "", "| metric | value |", "|---|---|"]
        for k, v in d.items():
            if k in ("kernel", "top_stalls"):
                continue
            lines.append(f"| {k} | {v} |")
        if t:
            lines.append(f"| DRAM GB/s (read+write / time) | {(rd + wr) / t / 1e9:.1f} |")
            if lts:
                lines.append(f"| L2 GB/s (lts__t_sectors x 32 B / time) | {lts / t / 1e9:.1f} |")
        lines.append(f"| top stall samples | {', '.join(f'{k}={v}' for k, v in d['top_stalls'].items())} |")
        lines.append("")
if not found:
    sys.exit(f"make_profiles: no prof_*_{tag}.ncu-rep[.gz] under gpurun_out/ -- refusing to overwrite the summaries")
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
open(os.path.join(ROOT, "profiles", f"ncu_summary_{tag}.md"), "w").write("\n".join(lines) + "\n")
json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)

lp = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
if os.path.exists(lp):
    rows = [r for r in csv.reader(open(lp)) if len(r) > 10]
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    data = [(r[ik], float(r[iv].replace(",", ""))) for r in rows[1:]]
    # the last step = every launch after the last L2-flush fill kernel (bench.py writes
    # a 256 MB buffer before each step)
    segs, cur = [], []
    for k, v in data:
        if "FillFunctor" in k:
            segs.append(cur)
            cur = []
        elif not k.startswith("void at::") and "::gather_kernel" not in k and "::stream_kernel" not in k:
            # (the flush's read-back reduction and the L2 probe are not step kernels)
            cur.append((k, v))
    segs.append(cur)
    # the last timed (flushed) step: the modal segment length is the step's launch count
    # (the warm-L2 steps that follow run without a flush, so they land in one segment)
    full = [sg for sg in segs if len(sg) >= 7]
    modal = max(set(len(sg) for sg in full), key=lambda n: sum(len(sg) == n for sg in full))
    step = [sg for sg in full if len(sg) == modal][-1]
    tot = sum(v for _, v in step)
    out = [f"# Launch list of one bench step ({tag})", "",
           "`ncu --metrics gpu__time_duration.sum --clock-control none` over `bench.py --steps 2 --warmup 3`; "
           "every launch of the last step (all libfg kernels).  Per-launch times are cold-cache and serialised: compare shares.", "",
           "| # | kernel | ns | share |", "|---|---|---|---|"]
    for i, (k, v) in enumerate(step):
        out.append(f"| {i} | `{k[:90]}` | {v:.0f} | {v / tot:.1%} |")
    out.append(f"| | total | {tot:.0f} | |")
    open(os.path.join(ROOT, "profiles", f"launches_{tag}.md"), "w").write("\n".join(out) + "\n")
print(json.dumps(traffic, indent=1)[:3000])
