"""Build development variants of libfg.so (kernel constants overridden with -D)
next to the product library, for A/B timing in one gpurun call:

    python tools/variants.py NAME=DEF1,DEF2 ...   -> paper_2008_11359_b200/lib/variants/libfg_NAME.so

Load one with FG_LIBFG=<path> (fg.py).  Experiments only; the product is
paper_2008_11359_b200/lib/libfg.so."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_11359_b200.build import build  # noqa: E402

for spec in sys.argv[1:]:
    name, _, defs = spec.partition("=")
    out = os.path.join(ROOT, "paper_2008_11359_b200", "lib", "variants", f"libfg_{name}.so")
    print(build(defines=[d for d in defs.split(",") if d], lib=out))
