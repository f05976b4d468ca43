"""GPU work curves (analysis.cpp:78-151) against the compiled reference's
work_curve / concavity_check: the trials of a batch size run as the parts of
one plan, each under its own plain stream, and the curve must equal the
reference's to the bit (|S^L| per trial is integer; mean / standard error
are summed in trial order). Mirrors proj/tests/test_analysis.cpp:67-167."""
import numpy as np
import pytest

import paper_2310_12403_b200 as cb
from oracle import oracle as O

pytestmark = pytest.mark.gpu

RW = 3


def need_ref():
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built")


@pytest.fixture(scope="module")
def plaw(gpu):
    need_ref()
    ref = O.generate_powerlaw(5000, 8, 0.6, 9)
    return cb.Graph.from_csr(ref.indptr, ref.indices), ref


def curve_array(c: cb.WorkCurve) -> np.ndarray:
    return np.array([[p.mean_sl, p.se_sl, p.work_per_seed, p.se_work] for p in c.points])


@pytest.mark.parametrize("kind,okind,k", [(cb.SamplerKind.kLabor0, O.LABOR0, 5),
                                          (cb.SamplerKind.kNs, O.NS, 4),
                                          (cb.SamplerKind.kFull, O.FULL, 1),
                                          (cb.SamplerKind.kRw, RW, 3)])
@pytest.mark.parametrize("per_launch", [1, 8, 64])
def test_work_curve_matches_reference(plaw, kind, okind, k, per_launch):
    g, ref = plaw
    sizes = [16, 64, 256, 1024]
    got = cb.work_curve(g, cb.SamplerConfig(kind, k), sizes, 20, 2, 4,
                        trials_per_launch=per_launch)
    want = O.work_curve_reference(ref, okind, k, sizes, 20, 2, 4)
    assert [p.batch_size for p in got.points] == sizes
    assert got.layer == 2
    assert np.array_equal(curve_array(got), want)


def test_work_curve_edge_mode_matches_reference(plaw):
    g, ref = plaw
    sizes = [4, 16, 64]
    got = cb.work_curve(g, cb.SamplerConfig(cb.SamplerKind.kLabor0, 5), sizes, 5, 2, 8,
                        cb.SeedMode.kEdge)
    want = O.work_curve_reference(ref, O.LABOR0, 5, sizes, 5, 2, 8, edge_mode=True)
    assert np.array_equal(curve_array(got), want)
    assert got.points[1].mean_sl > got.points[0].mean_sl


def test_work_curve_toy6_edge_mode(gpu):
    """test_analysis.cpp:116-134 on toy6 (s <- s+1, s <- s+2 mod 6)."""
    need_ref()
    src = [(s + d) % 6 for s in range(6) for d in (1, 2)]
    dst = [s for s in range(6) for _ in (1, 2)]
    ref = O.build_csr(src, dst, 6, impl="reference")
    g = cb.Graph.from_csr(ref.indptr, ref.indices)
    cfg = cb.SamplerConfig()
    with pytest.raises(cb.InputError):
        cb.work_curve(g, cfg, [7], 2, 1, 0)
    with pytest.raises(cb.InputError):
        cb.work_curve(g, cfg, [4, 4], 2, 1, 0)
    with pytest.raises(cb.InputError):
        cb.work_curve(g, cfg, [4], 0, 1, 0)
    got = cb.work_curve(g, cfg, [4, 12], 5, 2, 8, cb.SeedMode.kEdge)
    want = O.work_curve_reference(ref, int(cfg.kind), cfg.fanout, [4, 12], 5, 2, 8, True)
    assert np.array_equal(curve_array(got), want)


def test_work_curve_saturates_on_ring(gpu):
    """test_analysis.cpp:67-79: FULL expansion of every vertex of a ring."""
    src = [i for i in range(12)] + [(i + 1) % 12 for i in range(12)]
    dst = [(i + 1) % 12 for i in range(12)] + [i for i in range(12)]
    ref = O.build_csr(src, dst, 12)
    g = cb.Graph.from_csr(ref.indptr, ref.indices)
    c = cb.work_curve(g, cb.SamplerConfig(cb.SamplerKind.kFull, 1), [12], 4, 3, 1)
    assert c.points[0].mean_sl == 12.0
    assert c.points[0].work_per_seed == 1.0
    assert c.points[0].se_sl == 0.0


def test_concavity_of_measured_labor_curve(plaw):
    """test_analysis.cpp:159-167, and the check equals the reference's."""
    g, ref = plaw
    sizes = [16, 32, 64, 128, 256, 512, 1024]
    c = cb.work_curve(g, cb.SamplerConfig(cb.SamplerKind.kLabor0, 5), sizes, 20, 2, 21)
    rep = cb.concavity_check(c)
    assert rep.passed
    d2, thr, vio, ok = O.concavity_check_reference(
        sizes, [p.mean_sl for p in c.points], [p.se_sl for p in c.points])
    assert ok == rep.passed
    assert np.array_equal(d2, [e.second_diff for e in rep.entries])
    assert np.array_equal(thr, [e.threshold for e in rep.entries])
    assert np.array_equal(vio, [e.violation for e in rep.entries])


def test_sample_multi_equals_separate_expands(plaw):
    """Part p of a multi-schedule batch equals expand() of the same seeds
    under schedule p (the trial-per-part layout changes nothing)."""
    g, _ = plaw
    cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, 5)
    rng = np.random.default_rng(3)
    seeds = [rng.choice(5000, size=s, replace=False).astype(np.uint32) for s in (100, 7, 0, 300)]
    scheds = [cb.SeedSchedule.plain(11 + i) for i in range(4)]
    pl = cb.Plan(g, None, 3, cfg, 300, parts=4)
    pl.sample_multi(seeds, scheds)
    for p in range(4):
        want = cb.expand(g, seeds[p], 3, cfg, scheds[p])
        for l in range(3):
            a, b = pl.block(p, l).as_dict(), want.blocks[l].as_dict()
            for key in ("dst", "src", "edges", "dst_pos"):
                assert np.array_equal(a[key], b[key]), (p, l, key)
    with pytest.raises(cb.InputError):  # no partition: cooperative mode refused
        pl.sample(seeds, scheds[0], cb.MODE_COOP)
    with pytest.raises(cb.InputError):  # mixed smoothing
        pl.sample_multi(seeds, scheds[:3] + [cb.SeedSchedule(4, 1, 2, 1)])
