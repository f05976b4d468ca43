"""GPU: the peer-memory cooperative step (dist.PeerCoop over cb_px_*): ranks
OR their src ids into the owners' exchange bitmaps through CUDA IPC
mappings, owners extract in place, requesters read ranks back, rows are
pulled from the owners' shards. The pool gives one GPU per call, so 2-3
processes share cuda:0 (IPC between processes on one device) and the
phase barrier is a host barrier over gloo; on a multi-GPU node the same
code maps peers over NVLink with an NCCL all-reduce as the barrier.
Results must equal the oracle's coop_sample bit for bit."""
import pytest

from tests.dist_harness import check_rank, spawn

pytestmark = pytest.mark.gpu


def _px_worker(rank, world, kind, fanouts, kappa, steps):
    import numpy as np

    import paper_2310_12403_b200 as cb
    from oracle import oracle as O
    from paper_2310_12403_b200.dist import PeerCoop, synth_shard

    n, m, gseed = 1 << 14, 1 << 17, 21
    g = cb.Graph.generate_rmat(n, m, gseed)
    ref = O.rmat(n, m, gseed)
    pm = cb.partition_random(g, world, 6)
    owner = pm.owner
    L, dim, dtype, fseed = len(fanouts), 24, "f16", 5
    store = synth_shard(g, pm, rank, dim, fseed, dtype)
    pc = PeerCoop(g, pm, rank, L, cb.SamplerConfig(cb.SamplerKind(kind), fanouts=fanouts),
                  max_seeds=4096, store=store)
    sched = cb.SeedSchedule.make(kappa, 8)
    for step in range(steps):  # consecutive batches reuse the exchange slots
        seeds = O.draw_coop_seeds(owner, world, 128, 6, step)
        pc.sample(seeds[rank], sched)
        pc.load_inputs()
        res, rows = pc.result(), pc.rows()
        exp = O.coop_sample(ref, owner, world, seeds, L, kind, fanouts,
                            O.Sched(sched.kappa, sched.z1, sched.z2, sched.iteration))
        check_rank(res, rows, exp, rank, world, L, fseed, dim, dtype)
        sched = cb.schedule_advance(sched)
    del np


@pytest.mark.parametrize("world,kind,fanouts,kappa,steps", [
    (2, 2, [10, 10, 10], 1, 3),
    (3, 1, [10, 5, 5], 1, 2),
    (2, 2, [25, 15], 4, 2),
])
def test_peer_coop(gpu, world, kind, fanouts, kappa, steps):
    spawn(world, _px_worker, (kind, fanouts, kappa, steps), timeout=600)
