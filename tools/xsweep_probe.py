"""L2 gather / stream bandwidth versus working-set size (libfgprobe.so
fgprobe_xsweep): does the random-row gather ceiling depend on how much of the
L2 the gathered X occupies?  Evidence for DESIGN.md §6 / §9.

    python tools/xsweep_probe.py > gpurun_out/xsweep.txt
"""
import ctypes
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = ctypes.CDLL(os.path.join(ROOT, "paper_2008_11359_b200", "lib", "libfgprobe.so"))
buf = torch.empty(200 << 20, dtype=torch.uint8, device="cuda")
buf.random_(0, 255)
torch.cuda.synchronize()
sizes = [4, 8, 16, 24, 32, 40, 48, 56, 64, 80, 96, 128, 160]
arr = (ctypes.c_int * len(sizes))(*sizes)
out = (ctypes.c_double * (2 * len(sizes)))()
rc = L.fgprobe_xsweep(ctypes.c_void_p(buf.data_ptr()), ctypes.c_int64(buf.numel()), arr, len(sizes), out, 1)
print("rc", rc)
if "--ld" in os.sys.argv or True:
    rc = L.fgprobe_ldmodes(ctypes.c_void_p(buf.data_ptr()), ctypes.c_int64(buf.numel()), 1)
    print("ldmodes rc", rc)
