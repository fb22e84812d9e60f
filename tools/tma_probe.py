"""TMA bulk-copy row gathers vs LDG row gathers on this GPU (libfgprobe.so):
the measurement behind DESIGN.md §9's TMA decision.

    python tools/tma_probe.py > gpurun_out/tma_probe.txt
"""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = ctypes.CDLL(os.path.join(ROOT, "paper_2008_11359_b200", "lib", "libfgprobe.so"))
buf = torch.empty(600 << 20, dtype=torch.uint8, device="cuda")
buf.random_(0, 255)
torch.cuda.synchronize()
out = (ctypes.c_double * 5)()
rc = L.fgprobe_l2_verbose(ctypes.c_void_p(buf.data_ptr()), ctypes.c_int64(buf.numel()), out, 1)
print("ldg gather ceilings:", [round(x, 1) for x in out], "rc", rc)
o4 = (ctypes.c_double * 4)()
rc = L.fgprobe_tma(ctypes.c_void_p(buf.data_ptr()), ctypes.c_int64(buf.numel()), o4, 1)
print("tma best: 2KiB %.1f / read %.1f ; 512B %.1f / read %.1f  rc %d" % (o4[0], o4[1], o4[2], o4[3], rc))
sys.stdout.flush()
o4 = (ctypes.c_double * 4)()
rc = L.fgprobe_gather4(ctypes.c_void_p(buf.data_ptr()), ctypes.c_int64(buf.numel()), o4, 1)
print("gather4 best: F128 %.1f / read %.1f ; F256 %.1f / read %.1f  rc %d" % (o4[0], o4[1], o4[2], o4[3], rc))
