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
