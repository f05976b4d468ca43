"""Randomised parity: many small random graphs (duplicate edges, self loops,
isolated vertices, hubs far above the fanout, degree exactly k) and random
configurations (sampler, fanouts per layer, L, kappa, P, seed lists with
repeats), GPU vs the compiled reference. Every case is seeded, so a failure
prints a reproducible case id."""
import numpy as np
import pytest

import paper_2310_12403_b200 as cb
from oracle import oracle as O

from .test_gpu_parity import assert_stack_eq, coop_eq, osched

pytestmark = pytest.mark.gpu

KINDS = [(cb.SamplerKind.kFull, O.FULL), (cb.SamplerKind.kNs, O.NS),
         (cb.SamplerKind.kLabor0, O.LABOR0), (cb.SamplerKind.kRw, 3)]
KAPPAS = [1, 3, 16, cb.KAPPA_INFINITY]


def random_csr(rng):
    n = int(rng.integers(1, 1500))
    m = int(rng.integers(0, 12 * n + 1))
    src = rng.integers(0, n, m)
    dst = rng.integers(0, n, m)
    if n > 2 and rng.random() < 0.7:  # a hub far above any fanout
        h = int(rng.integers(0, n))
        extra = int(rng.integers(50, 400))
        src = np.concatenate([src, rng.integers(0, n, extra)])
        dst = np.concatenate([dst, np.full(extra, h)])
    return O.build_csr(src, dst, n, impl="reference")


def random_case(case: int):
    rng = np.random.default_rng(1000 + case)
    ref = random_csr(rng)
    kind, okind = KINDS[int(rng.integers(0, len(KINDS)))]
    L = int(rng.integers(1, 4))
    fanouts = [int(rng.integers(1, 12)) for _ in range(L)]
    kappa = KAPPAS[int(rng.integers(0, len(KAPPAS)))]
    sched = cb.SeedSchedule.make(kappa, int(rng.integers(0, 1 << 40)))
    for _ in range(int(rng.integers(0, 5))):
        sched = cb.schedule_advance(sched)
    return rng, ref, kind, okind, L, fanouts, sched


@pytest.mark.parametrize("case", range(64))
def test_fuzz_expand(gpu, case):
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built")
    rng, ref, kind, okind, L, fanouts, sched = random_case(case)
    g = cb.Graph.from_csr(ref.indptr, ref.indices)
    ns = int(rng.integers(0, min(ref.n, 300) + 1))
    seeds = rng.integers(0, ref.n, ns).astype(np.uint32)  # repeats allowed
    cfg = cb.SamplerConfig(kind, fanouts=fanouts)
    got = cb.expand(g, seeds, L, cfg, sched)
    want = O.expand(ref, seeds, L, okind, fanouts, osched(sched), impl="reference")
    assert_stack_eq(got, want, f"case {case}: n={ref.n} m={ref.m} {kind.name} L={L} "
                               f"k={fanouts} kappa={sched.kappa}")


@pytest.mark.parametrize("case", range(32))
def test_fuzz_coop(gpu, case):
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built")
    rng, ref, kind, okind, L, fanouts, sched = random_case(100 + case)
    if kind == cb.SamplerKind.kRw:
        kind, okind = cb.SamplerKind.kLabor0, O.LABOR0
    if ref.n < 4:
        pytest.skip("graph too small to partition")
    fanouts = [fanouts[0]] * L  # the reference's coop_sample takes one fanout
    P = int(rng.integers(2, 6))
    g = cb.Graph.from_csr(ref.indptr, ref.indices)
    pm = cb.partition_random(g, P, case)
    owner = O.partition_random(ref.n, P, case)
    members = [np.nonzero(owner == p)[0].astype(np.uint32) for p in range(P)]
    seeds = [rng.choice(mb, size=int(rng.integers(0, min(len(mb), 60) + 1)), replace=False)
             .astype(np.uint32) if len(mb) else np.zeros(0, np.uint32) for mb in members]
    res = cb.coop_sample(g, pm, seeds, L, cb.SamplerConfig(kind, fanouts[0]), sched)
    exp = O.coop_sample(ref, owner, P, seeds, L, okind, fanouts[0], osched(sched),
                        impl="reference")
    coop_eq(res, exp, P, L, f"case {case}: n={ref.n} P={P} {kind.name} L={L} k={fanouts[0]} "
                            f"kappa={sched.kappa}")
