"""GPU: smoothed-variate decisions inside the guard band are resolved on the
host with the reference's own arithmetic (VariateSource::finish,
samplers.hpp:96-100; rng.cpp:7-52), so smoothed sampling is the reference's
by construction, not by luck.

The guard band is widened (1e-12 -> 1e-3 .. 1e-2) so thousands of decisions
land in it; `perturb` makes the device decide every unresolved in-band case
WRONGLY, so the batch is only correct if the host's exact values are fed back
and the batch re-sampled. Results must equal the oracle bit for bit, and the
asynchronous path must refuse (UncertifiedError) rather than return a batch
with unresolved decisions."""
import numpy as np
import pytest

import paper_2310_12403_b200 as cb
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def osched(s):
    return O.Sched(s.kappa, s.z1, s.z2, s.iteration)


def stack_eq(got, want, where):
    for l, (a, b) in enumerate(zip(got.blocks, want)):
        d = a.as_dict()
        for k in ("dst", "src", "edges", "dst_pos"):
            assert np.array_equal(d[k], b[k]), f"{where} layer {l} {k} differs"


@pytest.fixture(scope="module")
def c1(gpu):
    n, m, seed = 1 << 16, 1 << 20, 42
    return cb.Graph.generate_rmat(n, m, seed), O.rmat(n, m, seed)


@pytest.mark.parametrize("kind,okind,band", [
    (cb.SamplerKind.kLabor0, O.LABOR0, 1e-3),
    (cb.SamplerKind.kLabor0, O.LABOR0, 1e-2),
    (cb.SamplerKind.kNs, O.NS, 1e-3),
])
@pytest.mark.parametrize("perturb", [False, True])
@pytest.mark.parametrize("n_seeds", [300, 3000])  # 3000: LABOR's per-vertex table path
def test_forced_in_band_decisions_are_resolved(c1, kind, okind, band, perturb, n_seeds):
    g, ref = c1
    cfg = cb.SamplerConfig(kind, 10)
    sched = cb.schedule_advance(cb.schedule_advance(cb.SeedSchedule.make(4, 77)))
    rng = np.random.default_rng(n_seeds)
    seeds = rng.choice(ref.n, n_seeds, replace=False).astype(np.uint32)
    pl = cb.Plan(g, None, 3, cfg, n_seeds)
    pl.set_guard(band, perturb=perturb)
    pl.sample([seeds], sched, cb.MODE_INDEP)
    resolved, reruns = pl.resolve_stats()
    assert resolved > 50, resolved  # the band really was hit
    if perturb:
        assert reruns >= 1  # every flipped decision had to be corrected
    for l in range(3):
        assert pl.layer_sizes(0, l)["uncertified"] == 0
    want = O.expand(ref, seeds, 3, okind, 10, osched(sched))
    stack_eq(pl.stack(0), want, f"{kind.name} band={band} perturb={perturb}")


def test_coop_parts_resolved(c1):
    """Cooperative P=3 (per-part keys): forced band + wrong device decisions."""
    g, ref = c1
    P = 3
    pm = cb.partition_random(g, P, 4)
    owner = O.partition_random(ref.n, P, 4)
    seeds = O.draw_coop_seeds(owner, P, 400, 4, 0)
    sched = cb.schedule_advance(cb.SeedSchedule.make(16, 3))
    cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, 10)
    pl = cb.Plan(g, pm, 3, cfg, 400)
    pl.set_guard(1e-3, perturb=True)
    pl.sample(seeds, sched, cb.MODE_COOP)
    resolved, reruns = pl.resolve_stats()
    assert resolved > 50 and reruns >= 1
    exp = O.coop_sample(ref, owner, P, seeds, 3, O.LABOR0, 10, osched(sched))
    for p in range(P):
        stack_eq(pl.stack(p), exp["stacks"][p], f"part {p}")


def test_async_path_refuses_unresolved(c1):
    """cb_sample (no host pass) with in-band decisions: strict mode raises on
    synchronize instead of handing out a possibly wrong batch; strict=False
    keeps the count visible; plain (unsmoothed) batches never record."""
    g, ref = c1
    cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, 10)
    seeds = np.arange(0, 6000, 3, dtype=np.uint32)
    pl = cb.Plan(g, None, 3, cfg, len(seeds))
    pl.set_guard(1e-2)
    sched = cb.schedule_advance(cb.SeedSchedule.make(4, 9))
    pl.sample([seeds], sched, cb.MODE_INDEP, sync=False)
    with pytest.raises(cb.UncertifiedError):
        pl.synchronize()
    pl.set_guard(1e-2, strict=False)
    pl.sample([seeds], sched, cb.MODE_INDEP, sync=False)
    pl.synchronize()
    assert sum(pl.layer_sizes(0, l)["uncertified"] for l in range(3)) > 0
    pl.set_guard(1e-2)
    pl.sample([seeds], cb.SeedSchedule.make(1, 9), cb.MODE_INDEP, sync=False)
    pl.synchronize()  # kappa = 1: plain variates, integer-exact, nothing to resolve
    # the default band at the synchronous entry: exact, nothing left over
    pl.set_guard()
    pl.sample([seeds], sched, cb.MODE_INDEP)
    want = O.expand(ref, seeds, 3, O.LABOR0, 10, osched(sched))
    stack_eq(pl.stack(0), want, "default band")
