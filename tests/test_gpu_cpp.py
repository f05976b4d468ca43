"""GPU: compile tests/cpp/test_shim.cpp against the C++ drop-in header and
run it (reference-style C++ test; checker = the compiled reference)."""
import os
import subprocess

import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin_shim(gpu, tmp_path):
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built")
    exe = tmp_path / "test_shim"
    libdir = os.path.join(ROOT, "paper_2310_12403_b200")
    refdir = os.path.join(ROOT, "oracle", "_ref")
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-I",
           os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests", "cpp", "test_shim.cpp"),
           "-L", libdir, "-lcoopbatch_b200", "-L", refdir, "-lcoopbatch_ref",
           f"-Wl,-rpath,{libdir}:{refdir}", "-o", str(exe)]
    subprocess.run(cmd, check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
