"""GPU: compute-sanitizer over a small workload that runs every kernel family
(tools/sanitize_run.py): memcheck (out-of-bounds / misaligned accesses),
racecheck (shared-memory hazards) and synccheck (barrier misuse) must report
no errors."""
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
    assert r.returncode == 0, tail
    assert "sanitize workload done" in r.stdout, tail
    out = r.stdout + r.stderr
    if tool == "racecheck":  # warnings (hazards) count as failures too
        assert "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out, tail
    else:
        assert "ERROR SUMMARY: 0 errors" in out, tail
