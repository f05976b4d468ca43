"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle on
identical graphs, seeds and RNG keys. Integer/index outputs must be
bit-identical; gathered rows must equal the oracle's values rounded once to
the table dtype (also bit-identical).

Mirrors the reference's own test strategy (proj/tests/test_samplers.cpp,
test_coop.cpp, acceptance.cpp c4/c9): block invariants, exact LABOR rule,
NS reservoir, union property / cooperative exactness, routing hand trace."""
import numpy as np
import pytest

import paper_2310_12403_b200 as cb
from oracle import oracle as O

pytestmark = pytest.mark.gpu

KINDS = [(cb.SamplerKind.kFull, O.FULL), (cb.SamplerKind.kNs, O.NS),
         (cb.SamplerKind.kLabor0, O.LABOR0)]


def osched(s: cb.SeedSchedule) -> O.Sched:
    return O.Sched(s.kappa, s.z1, s.z2, s.iteration)


def assert_stack_eq(got: cb.LayerStack, want: list, where=""):
    assert len(got.blocks) == len(want)
    for l, (a, b) in enumerate(zip(got.blocks, want)):
        d = a.as_dict()
        for k in ("dst", "src", "edges", "dst_pos"):
            assert d[k].shape == b[k].shape, f"{where} layer {l} {k} shape {d[k].shape} vs {b[k].shape}"
            assert np.array_equal(d[k], b[k]), f"{where} layer {l} {k} differs"


@pytest.fixture(scope="module")
def c1(gpu):
    """Config 1: R-MAT 2^16 vertices, 2^20 edges (avg degree 16)."""
    n, m, seed = 1 << 16, 1 << 20, 42
    g = cb.Graph.generate_rmat(n, m, seed)
    return g, O.rmat(n, m, seed)


@pytest.fixture(scope="module")
def powerlaw(gpu):
    ref = O.generate_powerlaw(3000, 9, 0.6, 5)
    return cb.Graph.from_csr(ref.indptr, ref.indices), ref


def test_rmat_csr_matches_oracle(c1):
    g, ref = c1
    indptr, indices = g.download()
    assert np.array_equal(indptr, ref.indptr)
    assert np.array_equal(indices, ref.indices)
    assert g.max_degree == int(np.diff(ref.indptr.astype(np.int64)).max())


def test_cbcs_roundtrip_with_reference(c1, tmp_path):
    """save_csr / load_csr (graph.cpp:216-252): a file written by the compiled
    reference loads into HBM unchanged, and a file written from HBM loads in
    the reference unchanged."""
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built")
    g, ref = c1
    O.save_csr_reference(ref, tmp_path / "ref.cbcs")
    h = cb.Graph.load_csr(str(tmp_path / "ref.cbcs"))
    ip, ix = h.download()
    assert np.array_equal(ip, ref.indptr) and np.array_equal(ix, ref.indices)
    assert h.max_degree == g.max_degree
    g.save_csr(str(tmp_path / "ours.cbcs"))
    back = O.load_csr_reference(tmp_path / "ours.cbcs")
    assert np.array_equal(back.indptr, ref.indptr) and np.array_equal(back.indices, ref.indices)
    assert (tmp_path / "ours.cbcs").read_bytes() == (tmp_path / "ref.cbcs").read_bytes()


def test_rmat_odd_sizes(gpu):
    for n, m, seed in [(1000, 5000, 1), (777, 3000, 9), (5, 12, 3)]:
        g = cb.Graph.generate_rmat(n, m, seed)
        ref = O.rmat(n, m, seed)
        ip, ix = g.download()
        assert np.array_equal(ip, ref.indptr) and np.array_equal(ix, ref.indices), (n, m)


@pytest.mark.parametrize("kind,okind", KINDS)
@pytest.mark.parametrize("kappa", [1, cb.KAPPA_INFINITY, 4])
def test_expand_parity_powerlaw(powerlaw, kind, okind, kappa):
    g, ref = powerlaw
    rng = np.random.default_rng(int(kind) * 7 + (kappa % 97))
    sched = cb.SeedSchedule.make(kappa, 99)
    for trial in range(4):
        seeds = rng.choice(ref.n, size=int(rng.integers(1, 200)), replace=False).astype(np.uint32)
        got = cb.expand(g, seeds, 3, cb.SamplerConfig(kind, 4), sched)
        want = O.expand(ref, seeds, 3, okind, 4, osched(sched))
        assert_stack_eq(got, want, f"{kind.name} kappa={kappa} trial={trial}")
        sched = cb.schedule_advance(sched)


@pytest.mark.parametrize("kind,okind", KINDS[1:])
def test_expand_parity_c1(c1, kind, okind):
    g, ref = c1
    owner = O.partition_random(ref.n, 1, 3)
    for step in range(3):
        seeds = O.draw_from_pool(np.arange(ref.n, dtype=np.uint32), 1024, 3, step)
        sched = cb.SeedSchedule.plain(O.hash_bits(3, [step]))
        got = cb.expand(g, seeds, 3, cb.SamplerConfig(kind, 10), sched)
        want = O.expand(ref, seeds, 3, okind, 10, osched(sched))
        assert_stack_eq(got, want, f"{kind.name} step={step}")
    del owner


def test_expand_matches_compiled_reference(powerlaw):
    """Spot-check against the reference's own compiled code (oracle/_ref)."""
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built")
    g, ref = powerlaw
    seeds = np.array([5, 9, 100, 317, 2999, 0, 1500], np.uint32)
    for kind, okind in KINDS:
        for kappa in (1, 4):
            sched = cb.SeedSchedule.make(kappa, 11)
            sched = cb.schedule_advance(cb.schedule_advance(sched))
            got = cb.expand(g, seeds, 3, cb.SamplerConfig(kind, 3), sched)
            want = O.expand(ref, seeds, 3, okind, 3, osched(sched), impl="reference")
            assert_stack_eq(got, want, f"{kind.name} kappa={kappa} vs reference")


def test_labor_inclusion_rule_star(gpu):
    """test_samplers.cpp:110-127 shape: hub with d=50, k=10 -> keep iff r<=0.2."""
    star = O.build_csr(np.arange(1, 51, dtype=np.uint32), np.zeros(50, np.uint32), 51)
    g = cb.Graph.from_csr(star.indptr, star.indices)
    for z in range(20):
        sched = cb.SeedSchedule.plain(1000 + z)
        got = cb.expand(g, [0], 1, cb.SamplerConfig(cb.SamplerKind.kLabor0, 10), sched)
        want = O.expand(star, [0], 1, O.LABOR0, 10, osched(sched))
        assert_stack_eq(got, want, f"z={z}")


def test_ns_reservoir_hub(gpu):
    """NS on a 5000-leaf star: slot-order emission of the reservoir."""
    star = O.build_csr(np.arange(1, 5001, dtype=np.uint32), np.zeros(5000, np.uint32), 5001)
    g = cb.Graph.from_csr(star.indptr, star.indices)
    for z in range(10):
        sched = cb.SeedSchedule.plain(z)
        got = cb.expand(g, [0, 3], 2, cb.SamplerConfig(cb.SamplerKind.kNs, 25), sched)
        want = O.expand(star, [0, 3], 2, O.NS, 25, osched(sched))
        assert_stack_eq(got, want, f"z={z}")
        assert got.blocks[0].num_edges() == 25


def test_edge_cases(powerlaw):
    g, ref = powerlaw
    cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, 5)
    # empty seeds
    got = cb.expand(g, np.zeros(0, np.uint32), 2, cfg, cb.SeedSchedule.plain(1))
    assert all(len(b.src_vertices) == 0 and b.num_edges() == 0 for b in got.blocks)
    # duplicate seeds at layer 0 (reference keeps them as distinct dsts)
    seeds = np.array([7, 7, 3, 7], np.uint32)
    got = cb.expand(g, seeds, 2, cfg, cb.SeedSchedule.plain(1))
    assert_stack_eq(got, O.expand(ref, seeds, 2, O.LABOR0, 5, O.plain_sched(1)), "dups")
    # isolated vertices only
    iso = np.flatnonzero(np.diff(ref.indptr.astype(np.int64)) == 0).astype(np.uint32)[:50]
    if len(iso):
        got = cb.expand(g, iso, 2, cfg, cb.SeedSchedule.plain(2))
        assert_stack_eq(got, O.expand(ref, iso, 2, O.LABOR0, 5, O.plain_sched(2)), "iso")
    with pytest.raises(cb.InputError):
        cb.expand(g, np.array([ref.n], np.uint32), 1, cfg, cb.SeedSchedule.plain(1))
    with pytest.raises(cb.InputError):
        cb.expand(g, [1], 0, cfg, cb.SeedSchedule.plain(1))
    with pytest.raises(cb.InputError):
        cb.expand(g, [1], 1, cb.SamplerConfig(cb.SamplerKind.kNs, 0), cb.SeedSchedule.plain(1))


def test_toy_routing_hand_trace(gpu):
    """test_coop.cpp:90-114: toy6, owners {0,0,0,1,1,1}, PE0 seeds {2}."""
    src = np.array([(s + 1) % 6 for s in range(6)] + [(s + 2) % 6 for s in range(6)], np.uint32)
    dst = np.array(list(range(6)) * 2, np.uint32)
    order = np.argsort(np.concatenate([np.arange(6) * 2, np.arange(6) * 2 + 1]), kind="stable")
    toy = O.build_csr(src[order], dst[order], 6)
    g = cb.Graph.from_csr(toy.indptr, toy.indices)
    pm = cb.partition_from_owner(g, [0, 0, 0, 1, 1, 1], 2)
    res = cb.coop_sample(g, pm, [[2], []], 1, cb.SamplerConfig(cb.SamplerKind.kFull, 1),
                         cb.SeedSchedule.plain(1))
    sc = res.exchanges[0].send_counts
    assert sc[0, 1] == 2 and sc[0, 0] == 1 and sc[1, 0] == 0
    assert res.exchanges[0].communicated(0) == 2
    assert res.owner_sets[0].tolist() == [2]
    assert res.owner_sets[1].tolist() == [3, 4]
    with pytest.raises(cb.InputError):
        cb.coop_sample(g, pm, [[3], []], 1, cb.SamplerConfig(), cb.SeedSchedule.plain(1))


def coop_eq(res: cb.CoopSampleResult, exp: dict, P: int, L: int, where=""):
    for p in range(P):
        assert_stack_eq(res.stacks[p], exp["stacks"][p], f"{where} part {p}")
        assert np.array_equal(res.owner_sets[p], exp["owner_sets"][p]), f"{where} owner_set {p}"
    for l in range(L):
        a, b = res.exchanges[l], exp["exchanges"][l]
        assert np.array_equal(a.send_counts, b["send_counts"]), f"{where} send_counts l={l}"
        assert np.array_equal(a.owner_row_counts, b["owner_row_counts"]), f"{where} orc l={l}"
        for p in range(P):
            assert np.array_equal(a.loc_part[p], b["loc_part"][p]), f"{where} loc_part {l},{p}"
            assert np.array_equal(a.loc_row[p], b["loc_row"][p]), f"{where} loc_row {l},{p}"


@pytest.mark.parametrize("kappa", [4, 64])
def test_smoothed_variate_table_c1(c1, kappa):
    """Smoothed LABOR where the scan space exceeds 2|V| (the per-vertex
    variate table path, samplers.cpp:114-129 memoisation) and where it does
    not (per-position evaluation): both bit-exact vs the oracle."""
    g, ref = c1
    cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, 10)
    sched = cb.schedule_advance(cb.SeedSchedule.make(kappa, 5))
    rng = np.random.default_rng(kappa)
    seeds = rng.choice(ref.n, 2000, replace=False).astype(np.uint32)
    pl = cb.Plan(g, None, 3, cfg, len(seeds))
    pl.sample([seeds], sched, cb.MODE_INDEP)
    scans = [pl.layer_sizes(0, l)["scan_total"] for l in range(3)]
    assert min(scans) < 2 * ref.n <= max(scans), scans  # both paths exercised
    want = O.expand(ref, seeds, 3, O.LABOR0, 10, osched(sched))
    assert_stack_eq(pl.stack(0), want, f"kappa={kappa}")


@pytest.mark.parametrize("P", [1, 2, 3, 5, 8])
def test_partition_members(c1, P):
    """partition.cpp:99-105 part_members: the shard layout of the feature
    tables (non-power-of-two part counts included)."""
    g, ref = c1
    for _ in range(3):  # the member sort once raced the owner copy
        pm = cb.partition_random(g, P, 11 + P)
        owner = O.partition_random(ref.n, P, 11 + P)
        assert np.array_equal(pm.owner, owner)
        for got, want in zip(pm.members(), O.part_members(owner, P)):
            assert np.array_equal(got, want)


@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("kind,okind", KINDS[1:])
def test_coop_parity_c1(c1, P, kind, okind):
    """acceptance.cpp c4: cooperative exactness for P in {2,4,8} (+ P=1)."""
    g, ref = c1
    pm = cb.partition_random(g, P, 17)
    owner = O.partition_random(ref.n, P, 17)
    assert np.array_equal(pm.owner, owner)
    for step in range(2):
        seeds = O.draw_coop_seeds(owner, P, 256, 17, step)
        sched = cb.SeedSchedule.make(1, 17 + step)
        res = cb.coop_sample(g, pm, seeds, 3, cb.SamplerConfig(kind, 10), sched)
        exp = O.coop_sample(ref, owner, P, seeds, 3, okind, 10, osched(sched))
        coop_eq(res, exp, P, 3, f"P={P} {kind.name} step={step}")


def test_step_metrics_match_reference_definitions(c1):
    """LayerMetrics / PeMetrics (coop.hpp:157-168) as coop_train_step fills
    them (coop.cpp:456-460, 541-546), from the oracle's coop_sample."""
    g, ref = c1
    P = 4
    pm = cb.partition_random(g, P, 23)
    owner = O.partition_random(ref.n, P, 23)
    seeds = O.draw_coop_seeds(owner, P, 100, 23, 0)
    sched = cb.SeedSchedule.plain(9)
    plan = cb.Plan(g, pm, 3, cb.SamplerConfig(cb.SamplerKind.kLabor0, 10), 100)
    plan.sample(seeds, sched, cb.MODE_COOP)
    got = cb.step_metrics(plan, cb.MODE_COOP, 400)
    exp = O.coop_sample(ref, owner, P, seeds, 3, O.LABOR0, 10, osched(sched))
    for p in range(P):
        for l in range(3):
            b = exp["stacks"][p][l]
            sc = exp["exchanges"][l]["send_counts"][p]
            want = (len(b["dst"]), len(b["src"]), len(b["edges"]), int(sc.sum() - sc[p]))
            m = got[p].layers[l]
            assert (m.s_l, m.s_tilde_l, m.e_l, m.comm_vertices) == want, (p, l)
        assert got[p].input_rows == len(exp["owner_sets"][p])
        assert got[p].feat_bytes == 400 * len(exp["owner_sets"][p])


@pytest.mark.parametrize("P", [2, 8])
def test_cross_edge_ratio_matches_reference(c1, P):
    """cross_edge_ratio (partition.cpp:79-89); random ownership cuts ~(P-1)/P
    of the edges (acceptance c6)."""
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built")
    g, ref = c1
    pm = cb.partition_random(g, P, 4)
    got = cb.cross_edge_ratio(g, pm)
    assert got == O.cross_edge_ratio_reference(ref, pm.owner, P)
    assert abs(got - (P - 1) / P) < 0.01


def test_coop_union_property(c1):
    """test_coop.cpp:128-157: cooperative input set == single-part union batch."""
    g, ref = c1
    P = 4
    pm = cb.partition_random(g, P, 5)
    owner = O.partition_random(ref.n, P, 5)
    seeds = O.draw_coop_seeds(owner, P, 128, 5, 0)
    sched = cb.SeedSchedule.plain(77)
    cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, 10)
    res = cb.coop_sample(g, pm, seeds, 3, cfg, sched)
    union = np.sort(np.concatenate(seeds))
    single = cb.expand(g, union, 3, cfg, sched)
    got = np.sort(np.concatenate(res.owner_sets))
    assert np.array_equal(got, single.input_vertices())


def test_coop_matches_compiled_reference(powerlaw):
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built")
    g, ref = powerlaw
    for P in (2, 4):
        pm = cb.partition_random(g, P, 3)
        owner = O.partition_random(ref.n, P, 3)
        seeds = O.draw_coop_seeds(owner, P, 40, 3, 1)
        for kind, okind in KINDS:
            sched = cb.SeedSchedule.make(4, 8)  # smoothed variates
            sched = cb.schedule_advance(sched)
            res = cb.coop_sample(g, pm, seeds, 3, cb.SamplerConfig(kind, 3), sched)
            exp = O.coop_sample(ref, owner, P, seeds, 3, okind, 3, osched(sched),
                                impl="reference")
            coop_eq(res, exp, P, 3, f"ref P={P} {kind.name}")


@pytest.mark.parametrize("dtype,dim", [("f32", 100), ("f16", 128), ("f32", 602), ("f64", 3)])
def test_gather_rows(c1, dtype, dim):
    g, ref = c1
    P = 4 if dtype == "f16" else 1
    pm = cb.partition_random(g, P, 9) if P > 1 else None
    owner = O.partition_random(ref.n, P, 9)
    seeds = O.draw_coop_seeds(owner, P, 200, 9, 0)
    store = cb.FeatureStore.synth(g, dim, 123, dtype, pm)
    cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, 10)
    sched = cb.SeedSchedule.plain(5)
    rows = cb.load_inputs(g, pm, seeds, 3, cfg, sched, store)
    exp = O.coop_sample(ref, owner, P, seeds, 3, O.LABOR0, 10, osched(sched))
    for p in range(P):
        ids = exp["stacks"][p][-1]["src"]
        want = O.feature_rows(123, dim, dtype, ids)
        assert rows[p].shape == want.shape
        assert np.array_equal(rows[p].view(np.uint8), want.view(np.uint8)), f"part {p}"


def test_gather_matches_reference_forward(powerlaw):
    """all_to_all_forward(load_rows(owner_sets)) of the compiled reference,
    cast once to f32, equals the fused device gather."""
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built")
    g, ref = powerlaw
    P, dim, seed = 4, 8, 31
    pm = cb.partition_random(g, P, seed)
    owner = O.partition_random(ref.n, P, seed)
    seeds = O.draw_coop_seeds(owner, P, 30, seed, 0)
    sched = cb.SeedSchedule.plain(4)
    store = cb.FeatureStore.synth(g, dim, seed, "f64", pm)
    rows = cb.load_inputs(g, pm, seeds, 2, cb.SamplerConfig(cb.SamplerKind.kLabor0, 4), sched,
                          store)
    exp, handle = O.coop_sample(ref, owner, P, seeds, 2, O.LABOR0, 4, osched(sched),
                                impl="reference", keep_handle=True)
    fs = O.RefFeatureStore(ref.n, dim, seed)
    owner_rows = [fs.load_rows(exp["owner_sets"][q]) for q in range(P)]
    flat = np.ascontiguousarray(np.concatenate(owner_rows))
    roff = np.zeros(P + 1, np.uint64)
    roff[1:] = np.cumsum([len(o) for o in exp["owner_sets"]])
    total = sum(len(exp["stacks"][p][-1]["src"]) for p in range(P))
    out = np.zeros((total, dim), np.float64)
    L = O.lib("reference")
    assert L.rf_all_to_all_forward(__import__("ctypes").byref(handle), 1, O._ptr(flat),
                                   O._ptr(roff), dim, O._ptr(out)) == 0
    O.coop_free_reference(handle)
    got = np.concatenate(rows)
    assert np.array_equal(got, out)


def test_coop_graph_replay_matches_oracle(c1):
    """A captured cooperative batch (P = 4: sampling, route / extract / locate
    rendezvous per layer, fused gather) replayed with new seeds and keys."""
    g, ref = c1
    P, b = 4, 128
    pm = cb.partition_random(g, P, 12)
    owner = O.partition_random(ref.n, P, 12)
    store = cb.FeatureStore.synth(g, 16, 2, "f32", pm)
    cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, 10)
    plan = cb.Plan(g, pm, 3, cfg, b)
    sched = cb.SeedSchedule.make(1, 21)
    seeds0 = O.draw_coop_seeds(owner, P, b, 12, 0)
    plan.sample(seeds0, sched, cb.MODE_COOP)
    plan.capture(np.arange(P + 1, dtype=np.uint64) * b, sched, cb.MODE_COOP, store)
    for step in range(1, 3):
        sched = cb.schedule_advance(sched)
        seeds = O.draw_coop_seeds(owner, P, b, 12, step)
        flat = np.ascontiguousarray(np.concatenate(seeds), dtype=np.uint32)
        plan.replay(flat.ctypes.data, sched, False, 3)
        plan.synchronize()
        exp = O.coop_sample(ref, owner, P, seeds, 3, O.LABOR0, 10, osched(sched))
        for p in range(P):
            assert_stack_eq(plan.stack(p), exp["stacks"][p], f"coop replay {step} part {p}")
            assert np.array_equal(plan.owner_set(p), exp["owner_sets"][p])
            rows = plan.rows(p, store)
            assert np.array_equal(rows, O.feature_rows(2, 16, "f32", exp["stacks"][p][-1]["src"]))


@pytest.mark.parametrize("kappa", [1, 4])
def test_graph_replay_matches_eager(c1, kappa):
    """cb_plan_capture/cb_plan_replay (the bench path) == eager batches."""
    g, ref = c1
    cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, 10)
    store = cb.FeatureStore.synth(g, 32, 3, "f32")
    plan = cb.Plan(g, None, 3, cfg, 512)
    pool = np.arange(ref.n, dtype=np.uint32)
    sched = cb.SeedSchedule.make(kappa, 5)
    seeds0 = O.draw_from_pool(pool, 512, 5, 0)
    plan.sample([seeds0], sched, cb.MODE_INDEP)
    plan.capture(np.array([0, 512], np.uint64), sched, cb.MODE_INDEP, store)
    # the sample + gather graph fuses the last relabel into the gather launch
    fresh = cb.Plan(g, None, 3, cfg, 8)
    with pytest.raises(cb.InputError):  # nothing captured yet
        fresh.captured_launches(3)
    per_layer = 4 if kappa == 4 else 3  # + the smoothed variate table
    assert plan.captured_launches(1) == 1 + 3 * per_layer + 1
    assert plan.captured_launches(2) == 1
    assert plan.captured_launches(3) == plan.captured_launches(1)
    for step in range(1, 4):
        sched = cb.schedule_advance(sched)
        seeds = O.draw_from_pool(pool, 512, 5, step)
        plan.replay(seeds.ctypes.data, sched, False, 3)
        plan.synchronize()
        got = plan.stack(0)
        want = O.expand(ref, seeds, 3, O.LABOR0, 10, osched(sched))
        assert_stack_eq(got, want, f"replay step {step}")
        rows = plan.rows(0, store)
        assert np.array_equal(rows, O.feature_rows(3, 32, "f32", want[-1]["src"]))


@pytest.mark.parametrize("kind,okind", KINDS[1:])
def test_expand_parity_large_sparse_bitmap(gpu, kind, okind):
    """n = 2^24 > 8.4M vertices: the dedup runs in summary-bitmap mode (only
    non-empty words visited). Checked against the oracle on the downloaded CSR."""
    n, m = 1 << 24, 1 << 25
    g = cb.Graph.generate_rmat(n, m, 77)
    ip, ix = g.download()
    ref = O.CSR(ip, ix)
    pool = np.arange(n, dtype=np.uint32)
    for step in range(2):
        seeds = O.draw_from_pool(pool, 2048, 77, step)
        sched = cb.SeedSchedule.make(1, 100 + step)
        got = cb.expand(g, seeds, 3, cb.SamplerConfig(kind, 10), sched)
        want = O.expand(ref, seeds, 3, okind, 10, osched(sched))
        assert_stack_eq(got, want, f"{kind.name} step={step}")


def test_coop_parity_large_sparse_bitmap(gpu):
    n, m, P = 1 << 24, 1 << 25, 4
    g = cb.Graph.generate_rmat(n, m, 78)
    ip, ix = g.download()
    ref = O.CSR(ip, ix)
    pm = cb.partition_random(g, P, 3)
    owner = O.partition_random(n, P, 3)
    seeds = O.draw_coop_seeds(owner, P, 512, 3, 0)
    sched = cb.SeedSchedule.plain(5)
    res = cb.coop_sample(g, pm, seeds, 3, cb.SamplerConfig(cb.SamplerKind.kLabor0, 10), sched)
    exp = O.coop_sample(ref, owner, P, seeds, 3, O.LABOR0, 10, osched(sched))
    coop_eq(res, exp, P, 3, "large coop")


@pytest.mark.parametrize("kappa", [1, 4])
def test_rw_sampler_matches_compiled_reference(powerlaw, kappa):
    """rw_block (samplers.cpp:202-285): random walks with restart, top-k by
    visit count (ties to the smaller id), through expand, vs the compiled
    reference with its default rw parameters (3 steps, p = 0.5, 100 walks)."""
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built")
    g, ref = powerlaw
    rng = np.random.default_rng(kappa)
    for trial in range(2):
        seeds = np.sort(rng.choice(ref.n, 150, replace=False)).astype(np.uint32)
        sched = cb.schedule_advance(cb.SeedSchedule.make(kappa, 40 + trial))
        got = cb.expand(g, seeds, 2, cb.SamplerConfig(cb.SamplerKind.kRw, 4), sched)
        want = O.expand(ref, seeds, 2, 3, 4, osched(sched), impl="reference")
        assert_stack_eq(got, want, f"RW kappa={kappa} trial={trial}")


def test_rw_sampler_c1_and_params(c1):
    """RW on the R-MAT config-1 graph (dead ends, hubs) and non-default
    parameters vs the compiled reference's sample_rw."""
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built")
    g, ref = c1
    rng = np.random.default_rng(5)
    seeds = np.sort(rng.choice(ref.n, 300, replace=False)).astype(np.uint32)
    sched = cb.SeedSchedule.plain(77)
    got = cb.expand(g, seeds, 3, cb.SamplerConfig(cb.SamplerKind.kRw, 10), sched)
    want = O.expand(ref, seeds, 3, 3, 10, osched(sched), impl="reference")
    assert_stack_eq(got, want, "RW c1")
    with pytest.raises(cb.InputError):
        cb.expand(g, seeds, 1, cb.SamplerConfig(cb.SamplerKind.kRw, 5, rw_walks=300, rw_length=3),
                  sched)


def test_repeated_seeds_beyond_edge_count(powerlaw):
    """Seeds may repeat (check_seeds, samplers.cpp:11-13 only bounds-checks):
    a layer-0 scan space larger than |E| overflows the first capacity plan on
    the device and is retried with a larger one; the result equals the
    oracle's."""
    g, ref = powerlaw
    deg = np.diff(ref.indptr.astype(np.int64))
    hubs = np.argsort(deg)[::-1][:3].astype(np.uint32)
    reps = int(3 * ref.m / max(1, int(deg[hubs].sum()))) + 1
    seeds = np.tile(hubs, reps)
    assert int(deg[seeds].sum()) > 2 * ref.m
    sched = cb.SeedSchedule.plain(3)
    for kind, okind in KINDS[1:]:
        got = cb.expand(g, seeds, 2, cb.SamplerConfig(kind, 4), sched)
        want = O.expand(ref, seeds, 2, okind, 4, osched(sched))
        assert_stack_eq(got, want, f"repeated {kind.name}")


def test_sample_labor0_caller_variate(powerlaw):
    """sample_labor0 with a caller variate (samplers.cpp:89-104, 305-312): the
    GPU block from the variate table equals the compiled reference's, with
    values exactly at k/d (inclusive), above 1 for low-degree dsts (rejected:
    no keep-all shortcut) and NaN (rejected)."""
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built")
    g, ref = powerlaw
    n = ref.n
    rng = np.random.default_rng(11)
    table = rng.random(n)
    deg = np.diff(ref.indptr.astype(np.int64))
    k = 4
    seeds = rng.choice(n, 300, replace=False).astype(np.uint32)
    # exact thresholds: the first neighbour of some dsts gets r = k / d
    for s in seeds[:40]:
        d = int(deg[s])
        if d:
            table[ref.indices[ref.indptr[s]]] = k / d
    table[rng.choice(n, 50, replace=False)] = 1.5
    table[rng.choice(n, 20, replace=False)] = np.nan
    for layer in (0, 2):
        got = cb.sample_labor0(g, seeds, k, table, layer)
        want = O.sample_labor0_reference(ref, seeds, k, table, layer)
        d = got.as_dict()
        for key in ("dst", "src", "edges", "dst_pos"):
            assert np.array_equal(d[key], want[key]), key
        assert got.layer == layer
    via_callable = cb.sample_labor0(g, seeds, k, lambda t: table[t])
    assert np.array_equal(via_callable.edges, got.edges)
    with pytest.raises(cb.InputError):
        cb.sample_labor0(g, seeds, 0, table)
    with pytest.raises(cb.InputError):
        cb.sample_labor0(g, seeds, k, table[:-1])


@pytest.mark.parametrize("layer", [0, 1, 3])
@pytest.mark.parametrize("kappa", [1, 4])
def test_sample_block_any_layer(powerlaw, layer, kappa):
    """sample_block (samplers.cpp:323-338) at layers > 0: the layer namespaces
    the variates (LABOR {2, layer}, NS {1, layer, s}, RW {3, layer, ...}); a
    1-layer plan with a layer base must equal the reference's block."""
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built")
    g, ref = powerlaw
    rng = np.random.default_rng(layer + 7 * kappa)
    seeds = rng.choice(ref.n, 200, replace=False).astype(np.uint32)
    sched = cb.SeedSchedule.make(kappa, 99)
    sched = cb.schedule_advance(cb.schedule_advance(sched))  # mid-group: smoothed for kappa 4
    for kind, okind, k in [(cb.SamplerKind.kLabor0, O.LABOR0, 5), (cb.SamplerKind.kNs, O.NS, 3),
                           (cb.SamplerKind.kRw, 3, 4)]:
        got = cb.sample_block(g, seeds, cb.SamplerConfig(kind, k), sched, layer).as_dict()
        want = O.sample_block(ref, seeds, okind, k, osched(sched), layer, impl="reference")
        for key in ("dst", "src", "edges", "dst_pos"):
            assert np.array_equal(got[key], want[key]), (kind, key)
        assert got["layer"] == layer
    if kappa == 1:
        ns = cb.sample_ns(g, seeds, 3, 1234, layer).as_dict()
        want = O.sample_block(ref, seeds, O.NS, 3, osched(cb.SeedSchedule.plain(1234)), layer,
                              impl="reference")
        assert np.array_equal(ns["edges"], want["edges"])


@pytest.mark.parametrize("kappa", [1, 4])
def test_rw_weighted_matches_compiled_reference(powerlaw, kappa):
    """RW on a weighted graph: pick_neighbor's weighted choice (samplers.cpp:
    139-165, cdf summed in f64 in CSR order, upper_bound of u * total) on the
    device vs the compiled reference's rw_block with Graph::weights set."""
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built")
    _, ref = powerlaw
    rng = np.random.default_rng(11 + kappa)
    w = rng.uniform(0.05, 4.0, ref.m).astype(np.float32)
    w[::7] = 1.0
    g = cb.Graph.from_csr(ref.indptr, ref.indices, weights=w)
    wref = O.CSR(ref.indptr, ref.indices, w)
    for trial in range(2):
        seeds = np.sort(rng.choice(ref.n, 120, replace=False)).astype(np.uint32)
        sched = cb.schedule_advance(cb.SeedSchedule.make(kappa, 90 + trial))
        cfg = cb.SamplerConfig(cb.SamplerKind.kRw, 5)  # reference defaults o=3, p=.5, a=100
        got = cb.expand(g, seeds, 2, cfg, sched)
        want = O.expand(wref, seeds, 2, 3, 5, osched(sched), impl="reference")
        assert_stack_eq(got, want, f"weighted RW kappa={kappa} trial={trial}")
