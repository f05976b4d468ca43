"""GPU: low-degree graphs, where labor_mark's tiles with record boundaries hold
more records than its shared-memory stage (1024 positions at average degree
~2 span ~500 records): the 32-record window walk, in the CTA-mode phase B
(small frontiers) and the warp-mode phase B (frontiers of >= 4.7K such
tiles). Stacks bit-exact vs the oracle (samplers.cpp:108-136, 340-354)."""
import numpy as np
import pytest

import paper_2310_12403_b200 as cb
from oracle import oracle as O

from .test_gpu_parity import assert_stack_eq, osched

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("logn,n_seeds", [(18, 3000), (22, 1 << 20)])
@pytest.mark.parametrize("kappa", [1, 4])
def test_low_degree_window_walk(gpu, logn, n_seeds, kappa):
    n, m, seed = 1 << logn, 1 << (logn + 1), 7
    g = cb.Graph.generate_rmat(n, m, seed)
    ref = O.rmat(n, m, seed)
    rng = np.random.default_rng(logn * 10 + kappa)
    sched = cb.SeedSchedule.make(kappa, 5)
    for trial in range(2):
        seeds = rng.choice(n, size=n_seeds, replace=False).astype(np.uint32)
        for fanout in (1, 3):  # below the typical degree: real keep decisions
            got = cb.expand(g, seeds, 3, cb.SamplerConfig(cb.SamplerKind.kLabor0, fanout), sched)
            want = O.expand(ref, seeds, 3, O.LABOR0, fanout, osched(sched))
            assert_stack_eq(got, want, f"2^{logn} kappa={kappa} k={fanout} trial={trial}")
        sched = cb.schedule_advance(sched)
