"""GPU: the multi-process cooperative step with the real per-part kernels
(CudaEngine over libcoopbatch_b200). Two ranks share cuda:0 (the pool gives one
GPU per call), ids/rows cross ranks through gloo with CPU staging — the same
DistCoop code drives NCCL on a multi-GPU box. Results must equal the oracle's
coop_sample bit for bit."""
import pytest

from tests.dist_harness import check_rank, spawn

pytestmark = pytest.mark.gpu


def _gpu_worker(rank, world, kind, fanouts, kappa):
    import numpy as np

    import paper_2310_12403_b200 as cb
    from oracle import oracle as O
    from paper_2310_12403_b200.dist import CudaEngine, DistCoop, synth_shard

    n, m, gseed = 1 << 14, 1 << 17, 21
    g = cb.Graph.generate_rmat(n, m, gseed)
    ref = O.rmat(n, m, gseed)
    pm = cb.partition_random(g, world, 6)
    owner = pm.owner
    seeds = O.draw_coop_seeds(owner, world, 128, 6, 2)
    L, dim, dtype, fseed = len(fanouts), 24, "f16", 5
    store = synth_shard(g, pm, rank, dim, fseed, dtype)
    eng = CudaEngine(g, pm, rank, L, cb.SamplerConfig(cb.SamplerKind(kind), fanouts=fanouts),
                     max_seeds=4096, store=store, comm_device="cpu")
    dc = DistCoop(eng)
    sched = cb.schedule_advance(cb.SeedSchedule.make(kappa, 8))
    res = dc.sample(seeds[rank], L, sched)
    rows = dc.load_inputs()
    exp = O.coop_sample(ref, owner, world, seeds, L, kind, fanouts,
                        O.Sched(sched.kappa, sched.z1, sched.z2, sched.iteration))
    check_rank(res, rows, exp, rank, world, L, fseed, dim, dtype)
    del np


@pytest.mark.parametrize("world,kind,fanouts,kappa", [
    (2, 2, [10, 10, 10], 1),
    (3, 1, [10, 5, 5], 1),
    (2, 2, [25, 15], 4),
])
def test_dist_coop_cuda_engine(gpu, world, kind, fanouts, kappa):
    spawn(world, _gpu_worker, (kind, fanouts, kappa), timeout=600)
