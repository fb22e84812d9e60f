"""Build libfg.so (the CUDA path) in-tree with nvcc for sm_100a.

    python -m paper_2008_11359_b200.build          # incremental
    python -m paper_2008_11359_b200.build --force

The .so lands in paper_2008_11359_b200/lib/ (git-ignored, shipped to the GPU
box by gpurun with the rest of the tree).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "lib", "libfg.so")
PROBE_SRC = os.path.join(PKG, "probe", "l2_probe.cu")
PROBE_LIB = os.path.join(PKG, "lib", "libfgprobe.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", f"-I{os.path.join(ROOT, 'include')}"]


def source_hash() -> str:
    """sha256 over everything libfg.so is built from (csrc sources and headers,
    include/fg.h, the nvcc arch and flags): the build identity that ncu captures
    under profiles/ are stamped with, so bench.py can refuse a stale capture."""
    import hashlib
    h = hashlib.sha256()
    files = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                   glob.glob(os.path.join(CSRC, "*.h"))) + [os.path.join(ROOT, "include", "fg.h")]
    for f in files:
        h.update(os.path.basename(f).encode())
        h.update(open(f, "rb").read())
    h.update(" ".join(ARCH + [x for x in FLAGS if not x.startswith("-I")]).encode())
    return h.hexdigest()[:16]


def _deps_mtime(src: str) -> float:
    hdrs = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "fg.h")]
    return max([os.path.getmtime(src)] + [os.path.getmtime(h) for h in hdrs])


def _compile(src: str, force: bool, defines=(), objdir: str = OBJ) -> tuple[str, str]:
    obj = os.path.join(objdir, os.path.basename(src) + ".o")
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= _deps_mtime(src):
        return obj, ""
    cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False, defines=(), lib: str | None = None) -> str:
    """Build libfg.so; `defines` / `lib` build a development VARIANT (kernel
    constants overridden with -D, objects under build/<tag>/) at another path --
    experiments only, never the product library (tools/variants.py)."""
    objdir = OBJ if not defines else os.path.join(OBJ, "v_" + "_".join(d.replace("=", "") for d in defines))
    out = LIB if lib is None else lib
    os.makedirs(objdir, exist_ok=True)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, force, defines, objdir), srcs))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                print(log, file=sys.stderr)
    if force or not os.path.exists(out) or os.path.getmtime(out) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", out, *objs, "-ldl"]
        subprocess.check_call(cmd)
    if lib is not None:
        return out
    # measurement utility for bench.py's roofline (L2 gather ceiling); not libfg
    if force or not os.path.exists(PROBE_LIB) or os.path.getmtime(PROBE_LIB) < os.path.getmtime(PROBE_SRC):
        subprocess.check_call([NVCC, *ARCH, "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "-o", PROBE_LIB,
                               PROBE_SRC])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
