"""CPU: the C++ drop-in library (libcoopbatch_core_b200.so) defines every
symbol the reference's replaced TUs (src/samplers.cpp, coop.cpp, cache.cpp)
define, so a program linked against the reference's coopbatch_core links
against it unchanged; and it resolves all of its own symbols (the
reference's kept TUs + our TUs + libcoopbatch_b200.so)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2310_12403_b200", "libcoopbatch_core_b200.so")
REF_OBJ = os.path.join(ROOT, "oracle", "_ref")


def _defined(path, dynamic):
    args = ["nm", "--defined-only", "-C"] + (["-D"] if dynamic else []) + [path]
    out = subprocess.run(args, capture_output=True, text=True, check=True).stdout
    syms = set()
    for line in out.splitlines():
        parts = line.split(" ", 2)
        if len(parts) == 3 and parts[1] in ("T", "W") and parts[2].startswith("coopbatch::") \
                and "(anonymous namespace)" not in parts[2]:
            syms.add(parts[2])
    return syms


def test_dropin_defines_the_replaced_tus():
    if not os.path.exists(LIB):
        pytest.skip("drop-in not built (needs the reference headers)")
    have = _defined(LIB, True)
    for tu in ("samplers", "coop", "cache"):
        obj = os.path.join(REF_OBJ, f"{tu}.o")
        if not os.path.exists(obj):
            pytest.skip("oracle/_ref objects not built")
        want = {s for s in _defined(obj, False) if "::~" not in s and "check_vertex" not in s}
        missing = sorted(want - have)
        assert not missing, f"{tu}.cpp symbols the drop-in lacks: {missing}"


def test_dropin_links_closed():
    if not os.path.exists(LIB):
        pytest.skip("drop-in not built (needs the reference headers)")
    r = subprocess.run(["ldd", "-r", LIB], capture_output=True, text=True)
    assert "undefined symbol" not in (r.stdout + r.stderr), r.stdout + r.stderr
    assert "libcoopbatch_b200.so" in r.stdout
