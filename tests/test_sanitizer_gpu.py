"""compute-sanitizer over every libfg entry point on small graphs:
memcheck (out-of-bounds / misaligned accesses), racecheck (shared-memory hazards),
synccheck (invalid barrier use)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(cuda_ok, tool):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not available")
    r = subprocess.run([cs, "--tool", tool, "--error-exitcode", "3", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_run.py")], capture_output=True, text=True, timeout=900)
    if r.returncode != 0 and "closed on this pool" in (r.stdout + r.stderr):
        # the pool's compute-sanitizer shim refuses to run (it has left GPUs needing a
        # reset); out-of-bounds writes are still caught by the parity tests' guard
        # regions (outputs pre-filled with NaN / garbage, exact sizes checked)
        pytest.skip("compute-sanitizer closed on this GPU pool")
    assert r.returncode == 0 and "sanitize_run: OK" in r.stdout, (r.stdout[-3000:] + r.stderr[-3000:])
