"""CPU: differential check of the plain-C restatement against the reference
compiled from its own sources (oracle/_ref), on randomized inputs — the
reference's own test strategy (test_coop.cpp union property, test_samplers
composability) applied to the checker itself. Skips where oracle/_ref is not
built."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.skipif(not O.available("reference"), reason="oracle/_ref not built")

KINDS = [O.FULL, O.NS, O.LABOR0]


def eq(a, b):
    if isinstance(a, dict):
        return all(eq(a[k], b[k]) for k in a)
    if isinstance(a, list):
        return len(a) == len(b) and all(eq(x, y) for x, y in zip(a, b))
    if isinstance(a, np.ndarray):
        return a.shape == b.shape and np.array_equal(a, b)
    return a == b


@pytest.fixture(scope="module")
def graphs():
    return [O.generate_powerlaw(1500, 7, 0.6, 11), O.generate_powerlaw(300, 25, 0.3, 2),
            O.rmat(1 << 11, 1 << 14, 3)]


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("kappa", [1, 3, O.KAPPA_INF])
def test_expand_random(graphs, kind, kappa):
    rng = np.random.default_rng(kind * 31 + kappa % 101)
    for g in graphs:
        rg = O.RefGraph(g)
        s = O.make_sched(kappa, int(rng.integers(1 << 30)))
        for _ in range(3):
            seeds = rng.integers(0, g.n, size=int(rng.integers(0, 60))).astype(np.uint32)
            fo = int(rng.integers(1, 12))
            a = O.expand(g, seeds, 3, kind, fo, s)
            b = O.expand(rg, seeds, 3, kind, fo, s, impl="reference")
            assert eq(a, b)
            s = O.advance(s)


def test_expand_per_layer_fanouts(graphs):
    g = graphs[0]
    rg = O.RefGraph(g)
    seeds = np.arange(0, 1500, 37, dtype=np.uint32)
    for kind in (O.NS, O.LABOR0):
        a = O.expand(g, seeds, 2, kind, [25, 15], O.plain_sched(4))
        b = O.expand(rg, seeds, 2, kind, [25, 15], O.plain_sched(4), impl="reference")
        assert eq(a, b)


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_coop_random(graphs, P):
    for gi, g in enumerate(graphs):
        rg = O.RefGraph(g)
        owner = O.partition_random(g.n, P, 5 + gi)
        assert np.array_equal(owner, O.partition_random(g.n, P, 5 + gi, "reference"))
        seeds = O.draw_coop_seeds(owner, P, 16, 5, gi)
        for kind in KINDS:
            for kappa in (1, 4):
                s = O.advance(O.make_sched(kappa, 9))
                a = O.coop_sample(g, owner, P, seeds, 3, kind, 4, s)
                b = O.coop_sample(rg, owner, P, seeds, 3, kind, 4, s, impl="reference")
                assert eq(a, b), (gi, kind, kappa)


def test_errors_match():
    g = O.generate_powerlaw(50, 3, 0.5, 1)
    rg = O.RefGraph(g)
    owner = O.partition_random(g.n, 2, 1)
    bad = [np.array([g.n], np.uint32)]
    for impl, gg in (("restated", g), ("reference", rg)):
        with pytest.raises(O.OracleError):
            O.expand(gg, bad[0], 1, O.NS, 3, O.plain_sched(1), impl=impl)
        with pytest.raises(O.OracleError):
            O.expand(gg, [1], 0, O.NS, 3, O.plain_sched(1), impl=impl)
        wrong = [np.flatnonzero(owner == 1)[:1].astype(np.uint32), np.zeros(0, np.uint32)]
        with pytest.raises(O.OracleError):
            O.coop_sample(gg, owner, 2, wrong, 1, O.NS, 3, O.plain_sched(1), impl=impl)


def test_build_csr_and_lru():
    rng = np.random.default_rng(3)
    src = rng.integers(0, 40, 300).astype(np.uint32)
    dst = rng.integers(0, 40, 300).astype(np.uint32)
    a = O.build_csr(src, dst, 40)
    b = O.build_csr(src, dst, 40, "reference")
    assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
    for cap in (1, 2, 7, 64):
        x, y = O.Lru(cap), O.Lru(cap, "reference")
        trace = rng.integers(0, 100, 3000)
        assert all(x.access(int(k)) == y.access(int(k)) for k in trace)
