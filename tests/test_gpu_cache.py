"""GPU: the device LRU feature cache (csrc/cache.cu) against the reference's
LruCache (cache.cpp:8-32, compiled in oracle/_ref) and its restatement, key by
key; feature_load_sim (cache.cpp:88-119) and run_dependent_experiment
(cache.cpp:137-208) against the compiled reference, step by step
(fingerprints, |S^L|, miss bytes, steady miss rate); rows served through the
cache (hits from HBM slots, misses from the table / host tier) equal the
oracle's rows."""
import numpy as np
import pytest

import paper_2310_12403_b200 as cb
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def ref_lru(cap):
    return O.Lru(cap, impl="reference" if O.available("reference") else "restated")


@pytest.mark.parametrize("cap,n,length,seed", [(1, 50, 400, 1), (7, 40, 3000, 2),
                                               (100, 300, 20000, 3), (500, 300, 5000, 4),
                                               (2000, 100000, 60000, 5)])
def test_lru_trace_matches_reference(gpu, cap, n, length, seed):
    rng = np.random.default_rng(seed)
    # skewed keys: many repeats, long distinct runs, and re-references
    keys = (rng.zipf(1.3, length) % n).astype(np.uint32)
    c = cb.LruCache(cap, n)
    got = c.access_trace(keys)
    r = ref_lru(cap)
    want = np.array([r.access(int(k)) for k in keys], np.uint8)
    assert np.array_equal(got, want)
    assert c.misses() == int(want.sum()) and c.hits() == length - int(want.sum())
    # resident set, most recent first
    seen, res = set(), []
    for k in keys[::-1]:
        if int(k) not in seen:
            seen.add(int(k))
            res.append(int(k))
    assert c.resident().tolist() == res[:cap]
    assert c.size() == min(cap, len(seen))


def test_lru_time_compaction(gpu):
    """Enough accesses to wrap the time bitmap several times."""
    n, cap = 64, 20
    rng = np.random.default_rng(9)
    c = cb.LruCache(cap, n)
    r = ref_lru(cap)
    for _ in range(30):
        keys = rng.permutation(n)[: rng.integers(1, n)].astype(np.uint32)
        got = c.access_trace(keys)
        want = np.array([r.access(int(k)) for k in keys], np.uint8)
        assert np.array_equal(got, want)


def test_lru_capacity_zero_rejected(gpu):
    with pytest.raises(cb.InputError):
        cb.LruCache(0, 10)


@pytest.fixture(scope="module")
def small(gpu):
    n, m, seed = 1 << 12, 1 << 15, 77
    return cb.Graph.generate_rmat(n, m, seed), O.rmat(n, m, seed)


@pytest.mark.parametrize("coop", [False, True])
def test_feature_load_sim_matches_restated(small, coop):
    g, ref = small
    P, L, b = 4, 2, 64
    pm = cb.partition_random(g, P, 3)
    owner = O.partition_random(ref.n, P, 3)
    cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, 5)
    steps, sched = [], cb.SeedSchedule.make(1, 5)
    for s in range(6):
        seeds = O.draw_coop_seeds(owner, P, b, 5, s)
        steps.append([cb.expand(g, seeds[p], L, cfg, sched) for p in range(P)])
        sched = cb.schedule_advance(sched)
    caches = [cb.LruCache(150, ref.n) for _ in range(P)]
    stats = cb.feature_load_sim(steps, caches, pm if coop else None, 16, 4)
    for p in range(P):
        lru = ref_lru(150)
        acc = miss = 0
        for si, step in enumerate(steps, start=1):
            for v in O.access_order(step[p].input_vertices(), O.hash_bits(si, [p])):
                if coop and owner[v] != p:
                    continue
                acc += 1
                miss += lru.access(int(v))
        assert (stats[p].accesses, stats[p].misses) == (acc, miss), p
        assert stats[p].bytes == miss * 16 * 4


@pytest.mark.parametrize("mode,kappa", [(cb.BatchMode.kSmoothed, 4), (cb.BatchMode.kNested, 4),
                                        (cb.BatchMode.kIndependent, 1),
                                        (cb.BatchMode.kSmoothed, cb.KAPPA_INFINITY)])
def test_dependent_experiment_matches_reference(small, mode, kappa):
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built")
    g, ref = small
    steps, cap, b, L, dim, bps, seed = 24, 600, 128, 2, 32, 2, 11
    got = cb.run_dependent_experiment(g, cb.MinibatchSchedule(mode, kappa, b), steps, cap,
                                      cb.SamplerConfig(cb.SamplerKind.kLabor0, 5), L, dim, bps,
                                      seed)
    want = O.dependent_experiment(ref, int(mode), kappa, b, steps, cap, O.LABOR0, 5, L, dim,
                                  bps, seed)
    assert [r.fingerprint for r in got.rows] == want["fingerprint"].tolist()
    assert [r.s_l for r in got.rows] == want["s_l"].tolist()
    assert [r.bytes for r in got.rows] == want["bytes"].tolist()
    assert got.steady_miss_rate == pytest.approx(want["steady"], abs=0, rel=0)


@pytest.mark.parametrize("host_tier", [False, True])
def test_cached_rows_match_oracle(small, host_tier):
    """Rows through the cache (hits from HBM slots, misses from the table)
    equal FeatureStore::load_rows at every step, with evictions."""
    g, ref = small
    dim, fseed = 24, 13
    store = cb.FeatureStore.synth(g, dim, fseed, "f32")
    if host_tier:
        store.set_tier(True)
    cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, 5)
    sizes = []

    def check(step, plan):
        ids = plan.block(0, 1).src_vertices
        sizes.append(len(ids))
        assert np.array_equal(plan.rows(0, store), O.feature_rows(fseed, dim, "f32", ids)), step

    res = cb.run_dependent_experiment(g, cb.MinibatchSchedule(cb.BatchMode.kSmoothed, 4, 96), 16,
                                      300, cfg, 2, dim, 4, 3, fingerprints=False, store=store,
                                      on_step=check)
    assert len(sizes) == 16 and max(sizes) > 300  # more rows than slots: evictions happen
    assert 0.0 < res.steady_miss_rate < 1.0
    if host_tier:
        store.set_tier(False)


def test_nested_batches(small):
    """nested_batches (cache.cpp:34-66): kappa b-sized slices of a super
    batch under one epoch seed, each contained layerwise in the super batch's
    expansion and equal to the oracle's expand of that slice."""
    g, ref = small
    rng = np.random.default_rng(2)
    sup = rng.choice(ref.n, 4 * 50, replace=False).astype(np.uint32)
    cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, 5)
    stacks = cb.nested_batches(g, sup, 4, 50, 2, cfg, 123)
    assert len(stacks) == 4
    for i, st in enumerate(stacks):
        want = O.expand(ref, sup[i * 50:(i + 1) * 50], 2, O.LABOR0, 5, O.plain_sched(123))
        for l in range(2):
            assert np.array_equal(st.blocks[l].src_vertices, want[l]["src"])
    with pytest.raises(cb.InputError):
        cb.nested_batches(g, sup[:199], 4, 50, 2, cfg, 123)


def test_clock_cache_rows_and_hit_rate(gpu):
    """The set-associative CLOCK cache over kappa-dependent batches: every row
    it serves equals the table's row (hits from its HBM slots, misses from the
    table in pinned host memory), and its hit rate is close to the exact LRU's
    of the same capacity on the same sequence."""
    import numpy as np

    n, m, seed = 1 << 15, 1 << 19, 11
    g = cb.Graph.generate_rmat(n, m, seed)
    store = cb.FeatureStore.synth(g, 24, 3, "f16")
    store.set_tier(True)
    cap = n // 8
    cc = cb.ClockCache(cap, store.row_bytes, ways=8)
    lru = cb.LruCache(cap, n, 0, 0)
    cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, 10)
    pl = cb.Plan(g, None, 2, cfg, 512)
    sched = cb.SeedSchedule.make(4, 5)
    rng = np.random.default_rng(2)
    pool = rng.choice(n, 2048, replace=False).astype(np.uint32)
    accesses = 0
    for step in range(16):
        seeds = pool[(step % 4) * 512:(step % 4 + 1) * 512]
        pl.sample([seeds], sched, cb.MODE_INDEP)
        cc.gather_plan(pl, 0, store)
        ids = pl.stack(0).input_vertices()
        want = O.feature_rows(3, 24, "f16", ids)
        assert np.array_equal(pl.rows(0, store).view(np.uint8), want.view(np.uint8)), step
        lru.access_ids(ids, cb.hash_bits(step, [0]))
        accesses += len(ids)
        sched = cb.schedule_advance(sched)
    h, ins, slots = cc.stats()
    assert slots == cap and 0 < h < accesses and ins <= accesses - h
    assert h >= 0.8 * lru.hits(), (h, lru.hits(), accesses)
    store.set_tier(False)
