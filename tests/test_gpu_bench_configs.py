"""GPU: bit-exact parity at the benchmark's own full-size configurations,
with the bench's seeds and schedules (bench.py CONFIGS / GRAPH_SEED /
RUN_SEED): the R-MAT CSR equals the oracle's generator, and the sampled
stacks, gathered rows and (c3) kappa-smoothed stacks equal the oracle's."""
import numpy as np
import pytest

import paper_2310_12403_b200 as cb
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def osched(s):
    return O.Sched(s.kappa, s.z1, s.z2, s.iteration)


@pytest.mark.parametrize("name,kappa", [("c2", 1), ("c3", 4)])
def test_bench_config_parity(gpu, name, kappa):
    import bench
    from paper_2310_12403_b200.seeds import draw_from_pool
    c = bench.CONFIGS[name]
    g = cb.Graph.generate_rmat(c["n"], c["m"], bench.GRAPH_SEED)
    ref = O.rmat(c["n"], c["m"], bench.GRAPH_SEED)
    ip, ix = g.download()
    assert np.array_equal(ip, ref.indptr) and np.array_equal(ix, ref.indices)
    L = len(c["fanouts"])
    store = cb.FeatureStore.synth(g, c["dim"], bench.FEAT_SEED, c["dtype"])
    pool = np.arange(c["n"], dtype=np.uint32)
    sched = cb.SeedSchedule.make(kappa, bench.RUN_SEED)
    for step in range(2):
        seeds = draw_from_pool(pool, c["batch"], bench.RUN_SEED, cb.hash_bits(step, [0]))
        cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, fanouts=c["fanouts"])
        rows = cb.load_inputs(g, None, [seeds], L, cfg, sched, store, cb.MODE_INDEP)[0]
        got = cb.expand(g, seeds, L, cfg, sched)
        want = O.expand(ref, seeds, L, O.LABOR0, c["fanouts"][0], osched(sched))
        for l in range(L):
            d = got.blocks[l].as_dict()
            for k in ("dst", "src", "edges", "dst_pos"):
                assert np.array_equal(d[k], want[l][k]), (name, step, l, k)
        ids = want[L - 1]["src"]
        pick = np.linspace(0, len(ids) - 1, 512).astype(np.int64)
        exp = O.feature_rows(bench.FEAT_SEED, c["dim"], c["dtype"], ids[pick])
        assert np.array_equal(rows[pick].view(np.uint8), exp.view(np.uint8)), (name, step)
        sched = cb.schedule_advance(sched)


def test_bench_config_parity_c4(gpu):
    """north_star's target, the bench headline: config 4 (papers100M-shaped,
    111M V / 1.6B E, 128 fp16 rows). The device CSR must match the digests of
    the oracle generator's CSR (tests/golden/c4_csr.json, make_c4_digest.py);
    then 2 steps x 1024 seeds of 3-layer LABOR-0 through the eager path and
    through the bench's captured sample + gather graph (fused relabel +
    gather launch), stacks and every gathered row vs the oracle."""
    import hashlib
    import json
    import os

    import bench
    from paper_2310_12403_b200.seeds import draw_from_pool
    with open(os.path.join(os.path.dirname(__file__), "golden", "c4_csr.json")) as f:
        gold = json.load(f)
    c = bench.CONFIGS["c4"]
    g = cb.Graph.generate_rmat(c["n"], c["m"], bench.GRAPH_SEED)
    ip, ix = g.download()
    assert hashlib.sha256(ip.tobytes()).hexdigest() == gold["indptr_sha256"]
    assert hashlib.sha256(ix.tobytes()).hexdigest() == gold["indices_sha256"]
    ref = O.CSR(ip, ix)  # == the oracle generator's CSR (digests above)
    del ip, ix
    L = len(c["fanouts"])
    store = cb.FeatureStore.synth(g, c["dim"], bench.FEAT_SEED, c["dtype"])
    cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, fanouts=c["fanouts"])
    pool = np.arange(c["n"], dtype=np.uint32)
    seeds = [draw_from_pool(pool, c["batch"], bench.RUN_SEED, cb.hash_bits(s, [0]))
             for s in range(3)]
    scheds = [cb.SeedSchedule.make(1, bench.RUN_SEED)]
    for _ in range(3):
        scheds.append(cb.schedule_advance(scheds[-1]))
    plan = cb.Plan(g, None, L, cfg, c["batch"])
    plan.sample([seeds[0]], scheds[0], cb.MODE_INDEP, sync=True)
    plan.capture(np.array([0, c["batch"]], np.uint64), scheds[0], cb.MODE_INDEP, store)

    def check(stack, rows, step, tag):
        want = O.expand(ref, seeds[step], L, O.LABOR0, c["fanouts"][0], osched(scheds[step]))
        for l in range(L):
            d = stack[l] if isinstance(stack, list) else stack.blocks[l].as_dict()
            for k in ("dst", "src", "edges", "dst_pos"):
                assert np.array_equal(d[k], want[l][k]), (tag, step, l, k)
        exp = O.feature_rows(bench.FEAT_SEED, c["dim"], c["dtype"], want[L - 1]["src"])
        assert np.array_equal(rows.view(np.uint8), exp.view(np.uint8)), (tag, step)

    for step in (1, 2):
        rows = cb.load_inputs(g, None, [seeds[step]], L, cfg, scheds[step], store,
                              cb.MODE_INDEP)[0]
        check(cb.expand(g, seeds[step], L, cfg, scheds[step]), rows, step, "eager")
        plan.replay(seeds[step].ctypes.data, scheds[step], False, 3)
        plan.synchronize()
        check(plan.stack(0), plan.rows(0, store), step, "captured")
