"""CPU, world_size 2 and 3 over gloo: the product's multi-process cooperative
orchestration (paper_2310_12403_b200.dist.DistCoop) reproduces the
reference's coop_sample exactly — per-rank blocks, send_counts rows,
src_location, owner sets — and the cooperative feature fetch returns the
requester-aligned rows of all_to_all_forward. Per-part compute is the
oracle (test infrastructure); the collectives and the exchange logic are the
product's."""
import numpy as np
import pytest

from tests.dist_harness import OracleEngine, check_rank, spawn


def _coop_worker(rank, world, kind, fanouts, kappa):
    from oracle import oracle as O
    from paper_2310_12403_b200 import SeedSchedule, schedule_advance
    from paper_2310_12403_b200.dist import DistCoop

    g = O.generate_powerlaw(800, 7, 0.6, 13) if O.available("reference") else O.rmat(1024, 6000, 13)
    owner = O.partition_random(g.n, world, 4)
    seeds = O.draw_coop_seeds(owner, world, 24, 4, 1)
    L, dim, dtype, fseed = len(fanouts), 6, "f32", 99
    eng = OracleEngine(g, owner, world, kind, fanouts, fseed, dim, dtype)
    dc = DistCoop(eng)
    sched = schedule_advance(SeedSchedule.make(kappa, 3))
    res = dc.sample(seeds[rank], L, sched)
    rows = dc.load_inputs()
    exp = O.coop_sample(g, owner, world, seeds, L, kind, fanouts,
                        O.Sched(sched.kappa, sched.z1, sched.z2, sched.iteration))
    check_rank(res, rows, exp, rank, world, L, fseed, dim, dtype)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind", [1, 2])  # NS, LABOR-0
def test_dist_coop_gloo(world, kind):
    spawn(world, _coop_worker, (kind, [5, 4, 3], 1))


def test_dist_coop_gloo_smoothed_per_layer_fanouts():
    spawn(2, _coop_worker, (2, [25, 15], 4))
