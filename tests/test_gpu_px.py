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


def _px_worker(rank, world, kind, fanouts, kappa, steps, barrier="device", captured=False,
               direct_rows=False):
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
                  max_seeds=4096, store=store, barrier=barrier, direct_rows=direct_rows)
    sched = cb.SeedSchedule.make(kappa, 8)
    for step in range(steps):  # consecutive batches reuse the exchange slots
        seeds = O.draw_coop_seeds(owner, world, 128, 6, step)
        if captured and step > 0:
            if step == 1:  # after one eager step on every rank
                pc.capture(len(seeds[rank]), sched)
            pc.step(seeds[rank], sched)  # one graph: L layers + barriers + rows
        else:
            pc.sample(seeds[rank], sched)
            pc.load_inputs()
        res, rows = pc.result(), pc.rows()
        exp = O.coop_sample(ref, owner, world, seeds, L, kind, fanouts,
                            O.Sched(sched.kappa, sched.z1, sched.z2, sched.iteration))
        check_rank(res, rows, exp, rank, world, L, fseed, dim, dtype)
        sched = cb.schedule_advance(sched)
    del np


@pytest.mark.parametrize("world,kind,fanouts,kappa,steps,barrier,direct", [
    (2, 2, [10, 10, 10], 1, 3, "device", False),
    (3, 1, [10, 5, 5], 1, 2, "device", True),   # rows read in place from peer shards
    (2, 2, [25, 15], 4, 2, "host", False),
])
def test_peer_coop(gpu, world, kind, fanouts, kappa, steps, barrier, direct):
    spawn(world, _px_worker, (kind, fanouts, kappa, steps, barrier, False, direct), timeout=600)


@pytest.mark.parametrize("world,kind,fanouts,kappa,steps", [
    (2, 2, [10, 10, 10], 1, 5),   # odd L: the two slot-parity graphs alternate
    (3, 2, [25, 15], 4, 4),       # even L, smoothed variates
    (2, 1, [10, 5, 5], 1, 3),     # NS
    (2, 2, [10], 1, 6),           # L = 1: four graphs before the slots realign
    (4, 2, [10, 10], 4, 3),       # four ranks
])
def test_peer_coop_captured(gpu, world, kind, fanouts, kappa, steps):
    """The whole cooperative step captured as one CUDA graph per rank (device
    barriers on IPC flags, no host in the layer loop), replayed over
    consecutive batches: bit-exact vs the oracle's coop_sample every step."""
    spawn(world, _px_worker, (kind, fanouts, kappa, steps, "device", True), timeout=600)


def _px_nccl_worker():
    import os

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2310_12403_b200 as cb
    from oracle import oracle as O
    from paper_2310_12403_b200.dist import PeerCoop, synth_shard

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda:0"))
    try:
        n, m, gseed = 1 << 13, 1 << 16, 5
        g = cb.Graph.generate_rmat(n, m, gseed)
        ref = O.rmat(n, m, gseed)
        pm = cb.partition_random(g, 1, 2)
        store = synth_shard(g, pm, 0, 16, 3, "f32")
        pc = PeerCoop(g, pm, 0, 3, cb.SamplerConfig(cb.SamplerKind.kLabor0, 10), 512, store,
                      barrier="nccl")
        seeds = O.draw_coop_seeds(pm.owner, 1, 256, 2, 0)
        sched = cb.SeedSchedule.plain(4)
        pc.sample(torch.from_numpy(seeds[0].view(np.int32)).cuda(), sched)  # device seeds
        pc.load_inputs()
        res, rows = pc.result(), pc.rows()
        exp = O.coop_sample(ref, pm.owner, 1, seeds, 3, O.LABOR0, 10,
                            O.Sched(sched.kappa, sched.z1, sched.z2, sched.iteration))
        from tests.dist_harness import check_rank
        check_rank(res, rows, exp, 0, 1, 3, 3, 16, "f32")
    finally:
        dist.destroy_process_group()
    del os


def test_peer_coop_nccl_single_rank(gpu):
    """The NCCL code paths of PeerCoop (handle all-gather over NCCL, the
    phase barrier as an NCCL all-reduce ordered on the plan stream, device
    seeds) at world size 1, the only NCCL world one GPU allows."""
    import torch

    from tests.dist_harness import free_port
    ctx = torch.multiprocessing.get_context("spawn")
    import os
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(free_port())
    p = ctx.Process(target=_px_nccl_worker)
    p.start()
    p.join(300)
    assert p.exitcode == 0


def _px_cache_worker(rank, world, kappa, steps, captured, host_tier, rcap=0):
    import paper_2310_12403_b200 as cb
    from oracle import oracle as O
    from paper_2310_12403_b200.dist import PeerCoop, synth_shard
    from tests.dist_harness import check_rank

    n, m, gseed = 1 << 14, 1 << 17, 21
    g = cb.Graph.generate_rmat(n, m, gseed)
    ref = O.rmat(n, m, gseed)
    pm = cb.partition_random(g, world, 6)
    owner = pm.owner
    L, dim, dtype, fseed, cap = 2, 24, "f16", 5, 600
    store = synth_shard(g, pm, rank, dim, fseed, dtype)
    cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, fanouts=[10, 10])
    pc = PeerCoop(g, pm, rank, L, cfg, max_seeds=4096, store=store)
    if host_tier:
        store.set_tier(True)  # misses cross the host link (the storage channel)
    pc.enable_cache(cap, rcap)
    lru = O.Lru(cap, impl="reference")  # the reference's LruCache, this owner's
    rlru = O.Lru(rcap, impl="reference") if rcap else None  # this requester's
    sched = cb.SeedSchedule.make(kappa, 8)
    # dependent minibatches: the same seeds every step, drifting variates
    seeds = O.draw_coop_seeds(owner, world, 96, 6, 0)
    total_h = 0
    for step in range(steps):
        if captured and step > 0:
            if step == 1:
                pc.capture(len(seeds[rank]), sched, rows=False)
            pc.step(seeds[rank], sched)
        else:
            pc.sample(seeds[rank], sched)
        key = cb.hash_bits(step + 1, [rank])  # feature_load_sim's key (cache.cpp:102)
        owned, hits, misses = pc.load_inputs_cached(key)
        res, rows = pc.result(), pc.rows()
        exp = O.coop_sample(ref, owner, world, seeds, L, O.LABOR0, 10,
                            O.Sched(sched.kappa, sched.z1, sched.z2, sched.iteration))
        check_rank(res, rows, exp, rank, world, L, fseed, dim, dtype)
        own = exp["owner_sets"][rank]
        want_m = sum(lru.access(int(v)) for v in O.access_order(own, key))
        assert owned == len(own) and misses == want_m and hits == len(own) - want_m, \
            (step, owned, hits, misses, len(own), want_m)
        total_h += hits
        if rlru is not None:  # rows of other owners through this requester's LRU
            src = exp["stacks"][rank][L - 1]["src"]
            remote = src[owner[src] != rank]
            rkey = cb.mix64(key ^ 0x5245515545)  # hstep(order_key, "REQUE")
            want_rm = sum(rlru.access(int(v)) for v in O.access_order(remote, rkey))
            nr, rh, rm = pc.requester_stats()
            assert nr == len(remote) and rm == want_rm and rh == nr - rm, \
                (step, nr, rh, rm, len(remote), want_rm)
            total_h += rh
        sched = cb.schedule_advance(sched)
    assert total_h > 0  # the dependent batches did reuse rows


@pytest.mark.parametrize("world,kappa,steps,captured,host_tier,rcap", [
    (2, 4, 5, False, False, 0),
    (3, 16, 4, True, True, 0),
    (2, 4, 5, True, False, 400),   # + requester-side cache
    (3, 64, 4, False, True, 300),
])
def test_peer_coop_owner_cache(gpu, world, kappa, steps, captured, host_tier, rcap):
    """The owner-side cached fetch: per step each owner's set goes through its
    LRU (hits/misses equal the reference LruCache fed access_order(S^L_q,
    hash_bits(step, {q})), feature_load_sim's loop, cache.cpp:100-110) and
    every rank's rows, pulled from the owners' staged rows, equal the
    oracle's -- with the shard in HBM or in the pinned host tier. With a
    requester-side cache the rows other ranks own go through a second LRU
    (the reference LruCache fed access_order(remote, hstep(key, tag)) must
    agree) and only its misses are pulled over peer memory."""
    spawn(world, _px_cache_worker, (kappa, steps, captured, host_tier, rcap), timeout=600)


def _px_clock_worker(rank, world, kappa, steps):
    import paper_2310_12403_b200 as cb
    from oracle import oracle as O
    from paper_2310_12403_b200.dist import PeerCoop, synth_shard
    from tests.dist_harness import check_rank

    n, m, gseed = 1 << 14, 1 << 17, 21
    g = cb.Graph.generate_rmat(n, m, gseed)
    ref = O.rmat(n, m, gseed)
    pm = cb.partition_random(g, world, 6)
    L, dim, dtype, fseed = 2, 24, "f16", 5
    store = synth_shard(g, pm, rank, dim, fseed, dtype)
    cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, fanouts=[10, 10])
    pc = PeerCoop(g, pm, rank, L, cfg, max_seeds=4096, store=store)
    store.set_tier(True)
    pc.enable_clock_cache(800)
    sched = cb.SeedSchedule.make(kappa, 8)
    seeds = O.draw_coop_seeds(pm.owner, world, 96, 6, 0)
    for step in range(steps):
        if step == 0:
            pc.sample(seeds[rank], sched)
            pc.load_inputs()
        else:
            if step == 1:
                pc.capture(len(seeds[rank]), sched)
            pc.step(seeds[rank], sched)  # sampling + cached row fetch in one graph
        res, rows = pc.result(), pc.rows()
        exp = O.coop_sample(ref, pm.owner, world, seeds, L, O.LABOR0, 10,
                            O.Sched(sched.kappa, sched.z1, sched.z2, sched.iteration))
        check_rank(res, rows, exp, rank, world, L, fseed, dim, dtype)
        sched = cb.schedule_advance(sched)
    hits, ins, _ = pc.ccache.stats()
    assert hits > 0 and ins > 0


def test_peer_coop_clock_cache_captured(gpu):
    """The owner-side CLOCK cache inside the captured step (shards in the host
    tier): rows bit-exact vs the oracle every step, and the dependent batches
    hit the cache."""
    spawn(2, _px_clock_worker, (4, 5), timeout=600)
