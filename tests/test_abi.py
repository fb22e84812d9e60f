"""C-ABI checks that need no GPU: libfg.so loads, exports every function
include/fg.h declares, and rejects bad arguments on the host before touching
the device (include/fg.h CONVENTIONS)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2008_11359_b200 import build, fg
    build.build()
    return fg.lib()


def header_functions():
    src = open(os.path.join(ROOT, "include", "fg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_]+\*?\s+\*?(fg_[a-z0-9_]+)\s*\(", src, flags=re.M)))


def test_exports_every_header_symbol(L):
    from paper_2008_11359_b200 import fg
    names = header_functions()
    assert len(names) >= 14, names
    assert sorted(names) == sorted(fg.SYMBOLS)
    for n in names:
        assert hasattr(L, n), f"libfg.so does not export {n}"


def test_abi_version_and_strings(L):
    assert L.fg_abi_version() == 1
    for s in range(8):
        assert L.fg_status_string(s).decode().startswith("FG_")
    assert b"unknown" in L.fg_status_string(99)


def test_host_validation_no_gpu(L):
    from paper_2008_11359_b200 import fg
    h = ctypes.c_void_p()
    assert L.fg_graph_create(4, 4, 0, None, None, None, 0, None, ctypes.byref(h)) == fg.FG_EINVAL
    assert b"row_ptr" in L.fg_last_error()
    assert L.fg_graph_create(4, 4, 0, ctypes.c_void_p(16), None, None, 0, None, None) == fg.FG_EINVAL
    assert L.fg_graph_create(-1, 4, 0, ctypes.c_void_p(16), None, None, 0, None, ctypes.byref(h)) == fg.FG_ESHAPE
    assert L.fg_spmm(None, 0, 0, 1, 4, None, None, None, 0, None, None, None, None, None, 0, None) == fg.FG_EINVAL
    assert L.fg_sddmm(None, 0, 1, 4, None, None, None, None) == fg.FG_EINVAL
    assert L.fg_edge_softmax(None, 1, None, None, None) == fg.FG_EINVAL
    assert L.fg_graph_destroy(None) == fg.FG_EINVAL
    assert L.fg_comm_init(None, 2, 0, ctypes.byref(h)) == fg.FG_EINVAL
    sz = ctypes.c_size_t(7)
    assert L.fg_spmm_workspace_size(None, 0, 0, 1, 4, 0, ctypes.byref(sz)) == fg.FG_EINVAL


def test_so_is_sm100a():
    """The shipped cubin targets sm_100a (cuobjdump lists the ELF arch)."""
    import shutil
    import subprocess
    from paper_2008_11359_b200 import fg
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", fg.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out, out[:500]


def test_probe_lib_loads_and_rejects_bad_args(L):
    """libfgprobe.so (bench.py's live L2-gather-ceiling probe) is built next to
    libfg.so, exports its entry point and rejects a too-small buffer before any
    launch."""
    path = os.path.join(ROOT, "paper_2008_11359_b200", "lib", "libfgprobe.so")
    P = ctypes.CDLL(path)
    P.fgprobe_l2.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_double)]
    out = (ctypes.c_double * 5)()
    assert P.fgprobe_l2(None, 0, out) != 0
    assert P.fgprobe_l2(ctypes.c_void_p(256), 1 << 20, out) != 0


def test_host_validation_new_entry_points_no_gpu(L):
    """fg_spmm_x16 / fg_sddmm_x16 / fg_sddmm_emul reject bad arguments on the
    host before any launch (include/fg.h)."""
    from paper_2008_11359_b200 import fg
    assert L.fg_spmm_x16(None, 0, 0, 1, 4, None, None, None, None, None, None) == fg.FG_EINVAL
    assert L.fg_sddmm_x16(None, 0, 1, 4, None, None, None, None) == fg.FG_EINVAL
    assert L.fg_sddmm_emul(None, 1, 4, None, None, None, None, None) == fg.FG_EINVAL
    assert b"NULL graph" in L.fg_last_error()
