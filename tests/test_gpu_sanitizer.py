"""GPU: compute-sanitizer over a small workload that runs every kernel family
(tools/sanitize_run.py): memcheck (out-of-bounds / misaligned accesses),
racecheck (shared-memory hazards) and synccheck (barrier misuse) must report
no errors. Where the GPU pool closes compute-sanitizer (its wrapper exits 86)
the sanitizer cases skip and test_sanitize_workload_plain runs the same
workload plainly (CUDA errors and the library's device flags raise through
the C-ABI)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(gpu, tool):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not found")
    r = subprocess.run([cs, "--tool", tool, "--error-exitcode", "3", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_run.py")],
                       capture_output=True, text=True, timeout=1500, cwd=ROOT)
    tail = (r.stdout + r.stderr)[-4000:]
    if r.returncode == 86 or "compute-sanitizer is closed" in tail:
        # the pool's compute-sanitizer wrapper refuses to run (exit 86)
        pytest.skip("compute-sanitizer closed on this GPU pool")
    assert r.returncode == 0, tail
    assert "sanitize workload done" in r.stdout, tail
    out = r.stdout + r.stderr
    if tool == "racecheck":  # warnings (hazards) count as failures too
        assert "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out, tail
    else:
        assert "ERROR SUMMARY: 0 errors" in out, tail


def test_sanitize_workload_plain(gpu):
    """The sanitizer workload without a sanitizer: every kernel family runs to
    completion with no CUDA error and no device error flag raised."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert "sanitize workload done" in r.stdout, tail
