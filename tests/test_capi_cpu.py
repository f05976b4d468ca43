"""CPU: the C-ABI boundary and the host-side mirror, without a GPU.

* libcoopbatch_b200.so loads and exports every entry point declared in
  include/coopbatch_cuda.h (no compute calls);
* the .so was built for sm_100a (cubin present);
* the host mirror's schedule / hash / seed-draw helpers equal the oracle's
  restatement of rng.cpp / cli.cpp.
"""
import ctypes
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O


def test_library_exports_every_header_symbol():
    from paper_2310_12403_b200 import _lib
    L = _lib.load()
    syms = _lib.header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert b"sm_100a" in L.cb_version()


def test_library_is_sm100a():
    from paper_2310_12403_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_device_is_a_clean_error():
    """Without a GPU the product fails loudly (status + message), never falls back."""
    from paper_2310_12403_b200 import _lib
    L = _lib.load()
    n = ctypes.c_int(-1)
    rc = L.cb_device_count(ctypes.byref(n))
    if rc == 0 and n.value > 0:
        pytest.skip("a GPU is visible")
    import paper_2310_12403_b200 as cb
    with pytest.raises((cb.CudaError, cb.InputError)):
        cb.Graph.generate_rmat(1 << 10, 1 << 12, 1)


def test_schedule_and_hash_mirror():
    import paper_2310_12403_b200 as cb
    for kappa in (1, 2, 7, cb.KAPPA_INFINITY):
        a = cb.SeedSchedule.make(kappa, 1234)
        b = O.make_sched(kappa, 1234)
        for _ in range(30):
            assert (a.kappa, a.z1, a.z2, a.iteration) == (b.kappa, b.z1, b.z2, b.iteration)
            a, b = cb.schedule_advance(a), O.advance(b)
    for ids in ([1], [2, 3, 4], [8, 1 << 40, 0]):
        assert cb.hash_bits(99, ids) == O.hash_bits(99, ids)
        assert cb.mix64(ids[-1]) == O.lib().ob_mix64(ids[-1])


def test_seed_draws_mirror():
    from paper_2310_12403_b200.seeds import coop_seeds, draw_from_pool
    owner = O.partition_random(5000, 4, 7)
    members = O.part_members(owner, 4)
    for step in range(3):
        a = coop_seeds(members, 64, 7, step)
        b = O.draw_coop_seeds(owner, 4, 64, 7, step)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))
    pool = np.arange(100, dtype=np.uint32)
    assert np.array_equal(draw_from_pool(pool, 100, 3, 5), O.draw_from_pool(pool, 100, 3, 5))
    with pytest.raises(ValueError):
        draw_from_pool(pool, 101, 3, 5)


def test_header_matches_loader_table():
    from paper_2310_12403_b200 import _lib
    assert set(_lib._SIGS) == set(_lib.header_symbols())


def test_build_artifacts_in_tree():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    assert os.path.exists(os.path.join(root, "paper_2310_12403_b200", "libcoopbatch_b200.so"))
    assert os.path.exists(os.path.join(root, "oracle", "liboracle.so"))


def test_cbcs_errors_before_any_device_work(tmp_path):
    """load_csr's error taxonomy (graph.cpp:231-284) through the C-ABI:
    IoError / FormatError / InputError map to CB_IO / CB_FORMAT / CB_INPUT,
    decided on the host before any device allocation."""
    import struct

    import paper_2310_12403_b200 as cb
    with pytest.raises(OSError) as e:
        cb.Graph.load_csr(str(tmp_path / "missing.cbcs"))
    assert "cannot open" in str(e.value)
    bad = tmp_path / "bad.cbcs"
    bad.write_bytes(b"XXXX" + b"\0" * 32)
    with pytest.raises(cb.FormatError):
        cb.Graph.load_csr(str(bad))
    trunc = tmp_path / "trunc.cbcs"
    trunc.write_bytes(b"CBCS" + struct.pack("<IQQ", 1, 3, 2) + struct.pack("<QQ", 0, 1))
    with pytest.raises(cb.FormatError, match="truncated"):
        cb.Graph.load_csr(str(trunc))
    ver = tmp_path / "ver.cbcs"
    ver.write_bytes(b"CBCS" + struct.pack("<I", 7))
    with pytest.raises(cb.FormatError, match="version"):
        cb.Graph.load_csr(str(ver))
    inv = tmp_path / "inv.cbcs"  # indices out of range -> validate_csr InputError
    inv.write_bytes(b"CBCS" + struct.pack("<IQQ", 1, 2, 1) + struct.pack("<QQQ", 0, 1, 1)
                    + struct.pack("<I", 5) + b"\0")
    with pytest.raises(cb.InputError, match="out of range"):
        cb.Graph.load_csr(str(inv))


def test_reference_cbcs_roundtrip_oracle(tmp_path):
    """The compiled reference's save_csr/load_csr (the fixture writer the GPU
    test reads back) round-trips a graph."""
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built")
    g = O.rmat(500, 3000, 4)
    O.save_csr_reference(g, tmp_path / "g.cbcs")
    h = O.load_csr_reference(tmp_path / "g.cbcs")
    assert np.array_equal(h.indptr, g.indptr) and np.array_equal(h.indices, g.indices)


def test_edge_pred_seeds_match_reference():
    """edge_pred_seeds (samplers.cpp:356-393): host seed generation of an
    edge-prediction batch equals the compiled reference."""
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built")
    from paper_2310_12403_b200.seeds import edge_pred_seeds
    g = O.rmat(2000, 16000, 8)
    rng = np.random.default_rng(3)
    src = rng.integers(0, g.n, 64)
    pos = np.array([(int(g.indices[g.indptr[v]]), v) if g.indptr[v + 1] > g.indptr[v]
                    else (v, (v + 1) % g.n) for v in src], dtype=np.uint32)
    for seed in (1, 99):
        got = edge_pred_seeds(g.indptr, g.indices, pos, seed)
        want = O.edge_pred_seeds_reference(g, pos, seed)
        assert np.array_equal(got, want)


def test_csv_report_format(tmp_path):
    """reports.py: `# key=value` header, column line, atomic write (cli.cpp:74-99)."""
    from paper_2310_12403_b200 import reports as R
    p = tmp_path / "cache.csv"
    R.write_csv(str(p), {"kappa": 4, "mode": "smoothed"}, R.CACHE_COLUMNS,
                [(0, 0.5, 10, 1280), (1, 0.25, 12, 768)])
    lines = p.read_text().splitlines()
    assert lines[:3] == ["# kappa=4", "# mode=smoothed", "step,miss_rate,s_l,bytes"]
    assert lines[3] == "0,0.5,10,1280" and not (tmp_path / "cache.csv.tmp").exists()
