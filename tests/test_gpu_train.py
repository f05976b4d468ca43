"""GPU: the GCN training step (f1; coop.cpp:161-357, 394-610) against the
compiled reference's coop_train_step / indep_train_step on the same graph,
seeds, schedule, FeatureStore and GcnModel::init weights. The device keeps
the reference's FP64 accumulation order, so the only differences are libm's
(tanh / exp / log): loss and gradients must agree to 1e-12 relative, far
inside the reference's own 1e-5 test tolerance (test_coop.cpp:362-393)."""
import numpy as np
import pytest

import paper_2310_12403_b200 as cb
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def osched(s):
    return O.Sched(s.kappa, s.z1, s.z2, s.iteration)


@pytest.fixture(scope="module")
def pl_graph(gpu):
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built")
    ref = O.generate_powerlaw(500, 8, 0.6, 77)
    return cb.Graph.from_csr(ref.indptr, ref.indices), ref


def rel_err(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def test_model_init_matches_reference_weights(pl_graph):
    g, ref = pl_graph
    m = cb.GcnModel.init(6, 5, 4, 2, 2)
    assert m.shape(0) == (5, 4) and m.shape(1) == (6, 5)
    # the reference's step with zero seeds would throw; compare through a step
    # whose gradient depends on every weight instead (see below)


@pytest.mark.parametrize("kind,okind", [(cb.SamplerKind.kFull, O.FULL),
                                        (cb.SamplerKind.kLabor0, O.LABOR0),
                                        (cb.SamplerKind.kNs, O.NS)])
@pytest.mark.parametrize("parts", [1, 2, 4])
def test_coop_train_step_matches_reference(pl_graph, kind, okind, parts):
    g, ref = pl_graph
    dim, classes, fseed, hidden, mseed, L = 6, 4, 1, 5, 2, 2
    batch = np.unique(np.array([cb.hash_bits(4, [i]) % ref.n for i in range(60)],
                               dtype=np.uint32))
    sched = cb.SeedSchedule.plain(31)
    model = cb.GcnModel.init(dim, hidden, classes, L, mseed)
    shapes = [model.shape(l) for l in range(L)]
    sizes = [r * c for r, c in shapes]
    if parts == 1:
        store = cb.FeatureStore.synth(g, dim, fseed, "f64")
        got = cb.indep_train_step(g, [batch], L, cb.SamplerConfig(kind, 4), sched, model, store,
                                  classes)
        loss, gw = O.train_step_reference(ref, 1, None, 1, [batch], L, okind, 4, osched(sched),
                                          dim, classes, fseed, hidden, mseed, sizes)
    else:
        pm = cb.partition_random(g, parts, 9)
        owner = pm.owner
        seeds = [batch[owner[batch] == p] for p in range(parts)]
        store = cb.FeatureStore.synth(g, dim, fseed, "f64", pm)
        got = cb.coop_train_step(g, pm, seeds, L, cb.SamplerConfig(kind, 4), sched, model, store,
                                 classes)
        loss, gw = O.train_step_reference(ref, 0, owner, parts, seeds, L, okind, 4,
                                          osched(sched), dim, classes, fseed, hidden, mseed,
                                          sizes)
    assert abs(got.loss - loss) <= 1e-12 * abs(loss)
    o = 0
    for l, (r, c) in enumerate(shapes):
        want = gw[o:o + r * c].reshape(r, c)
        o += r * c
        assert rel_err(got.grad_w[l], want) < 1e-12, (l, rel_err(got.grad_w[l], want))


def test_indep_multi_part_and_three_layers(pl_graph):
    g, ref = pl_graph
    dim, classes, fseed, hidden, mseed, L = 5, 3, 8, 7, 3, 3
    rng = np.random.default_rng(1)
    seeds = [np.sort(rng.choice(ref.n, 40, replace=False)).astype(np.uint32) for _ in range(3)]
    sched = cb.schedule_advance(cb.SeedSchedule.make(4, 6))  # smoothed variates
    model = cb.GcnModel.init(dim, hidden, classes, L, mseed)
    sizes = [r * c for r, c in (model.shape(l) for l in range(L))]
    store = cb.FeatureStore.synth(g, dim, fseed, "f64")
    got = cb.indep_train_step(g, seeds, L, cb.SamplerConfig(cb.SamplerKind.kLabor0, 3), sched,
                              model, store, classes)
    loss, gw = O.train_step_reference(ref, 1, None, 3, seeds, L, O.LABOR0, 3, osched(sched), dim,
                                      classes, fseed, hidden, mseed, sizes)
    assert abs(got.loss - loss) <= 1e-12 * abs(loss)
    flat = np.concatenate([x.ravel() for x in got.grad_w])
    assert rel_err(flat, gw) < 1e-12


def test_coop_equals_union_batch_indep(pl_graph):
    """test_coop.cpp:362-393: the cooperative step equals the single-part
    step on the union batch (loss and gradients within 1e-5)."""
    g, ref = pl_graph
    batch = np.unique(np.array([cb.hash_bits(4, [i]) % ref.n for i in range(60)],
                               dtype=np.uint32))
    sched = cb.SeedSchedule.plain(31)
    model = cb.GcnModel.init(6, 5, 4, 2, 2)
    cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, 4)
    one = cb.indep_train_step(g, [batch], 2, cfg, sched, model,
                              cb.FeatureStore.synth(g, 6, 1, "f64"), 4)
    for parts in (2, 4):
        pm = cb.partition_random(g, parts, 9)
        seeds = [batch[pm.owner[batch] == p] for p in range(parts)]
        co = cb.coop_train_step(g, pm, seeds, 2, cfg, sched, model,
                                cb.FeatureStore.synth(g, 6, 1, "f64", pm), 4)
        assert abs(co.loss - one.loss) / abs(one.loss) < 1e-5
        for a, b in zip(co.grad_w, one.grad_w):
            assert rel_err(a, b) < 1e-5
