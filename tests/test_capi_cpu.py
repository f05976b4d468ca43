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


def test_first_distinct_equals_sequential_rejection():
    """seeds.first_distinct (vectorised) == the reference's sequential
    rejection loop (cli.cpp:121-139, analysis.cpp:15-31) restated here."""
    from paper_2310_12403_b200.coopbatch import hash_bits, hash_uniform
    from paper_2310_12403_b200.seeds import first_distinct
    for space, count, seed, tag in [(100, 10, 5, 7), (12, 12, 1, 3), (5000, 1024, 4, 99),
                                    (1, 1, 0, 0), (50, 0, 2, 2)]:
        want, seen, a = [], set(), 0
        while len(want) < count:
            u = hash_uniform(seed, [8, tag, a])
            a += 1
            v = min(int(u * float(space)), space - 1)
            if v not in seen:
                seen.add(v)
                want.append(v)
        got = first_distinct(hash_bits(seed, [8, tag]), space, count)
        assert got.tolist() == want


def test_concavity_check_matches_reference():
    """analysis.concavity_check == the compiled reference's (analysis.cpp:126-151)."""
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built")
    from paper_2310_12403_b200.analysis import (WorkCurve, WorkCurvePoint,
                                                concavity_check)
    from paper_2310_12403_b200.coopbatch import InputError
    rng = np.random.default_rng(0)
    cases = [([64, 128, 256, 512], [640.0, 1280, 2560, 5120], [0.0] * 4),
             ([64, 128, 256, 512], [0.001 * b * b for b in (64, 128, 256, 512)], [0.0] * 4)]
    for _ in range(20):
        b = np.cumsum(rng.integers(1, 100, 6)).tolist()
        cases.append((b, np.sqrt(np.array(b, float) * 50).tolist(), rng.random(6).tolist()))
    for sizes, mean, se in cases:
        c = WorkCurve(3, [WorkCurvePoint(s, m, e) for s, m, e in zip(sizes, mean, se)])
        rep = concavity_check(c)
        d2, thr, vio, ok = O.concavity_check_reference(sizes, mean, se)
        assert rep.passed == ok
        assert [e.second_diff for e in rep.entries] == d2.tolist()
        assert [e.threshold for e in rep.entries] == thr.tolist()
        assert [e.violation for e in rep.entries] == vio.tolist()
    with pytest.raises(InputError):
        concavity_check(WorkCurve(3, [WorkCurvePoint(1), WorkCurvePoint(2)]))


def test_draw_batch_and_split_by_owner():
    """acceptance.cpp:64-83 restated: draw_batch's {31337, attempt} rejection
    stream and split_by_owner's order-preserving split."""
    from paper_2310_12403_b200.coopbatch import hash_uniform
    from paper_2310_12403_b200.seeds import draw_batch, split_by_owner
    for n, count, seed in [(2000, 128, 17), (10, 10, 3), (5, 1, 0)]:
        want, seen, a = [], set(), 0
        while len(want) < count:
            v = min(int(hash_uniform(seed, [31337, a]) * float(n)), n - 1)
            a += 1
            if v not in seen:
                seen.add(v)
                want.append(v)
        assert draw_batch(n, count, seed).tolist() == want
    owner = np.array([0, 1, 1, 0, 2, 2, 1], np.uint32)
    parts = split_by_owner([6, 0, 4, 1, 3, 5], owner, 3)
    assert [p.tolist() for p in parts] == [[0, 3], [6, 1], [4, 5]]


def test_csv_curve_and_partition_formats(tmp_path):
    """cli.cpp:153-188: curve header names the layer count, doubles print like
    std::ostream (%g, 6 significant digits), partition rows are vertex,part."""
    from paper_2310_12403_b200 import reports as R
    from paper_2310_12403_b200.analysis import WorkCurve, WorkCurvePoint
    c = WorkCurve(2, [WorkCurvePoint(64, 1234.5678901, 0.0001234567, 19.29012328),
                      WorkCurvePoint(128, 2e7, 1e-7, 156250.0)])
    p = tmp_path / "curve.csv"
    R.write_csv(str(p), {"layers": 2}, R.curve_columns(2), R.curve_rows(c))
    lines = p.read_text().splitlines()
    assert lines[1] == "batch_size,mean_s2,se_s2,work_per_seed"
    assert lines[2] == "64,1234.57,0.000123457,19.2901"
    assert lines[3] == "128,2e+07,1e-07,156250"
    q = tmp_path / "part.csv"
    R.write_csv(str(q), {"parts": 2}, R.PARTITION_COLUMNS, R.partition_rows(np.array([1, 0, 1])))
    assert q.read_text().splitlines()[1:] == ["vertex,part", "0,1", "1,0", "2,1"]
