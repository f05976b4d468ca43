"""kappa sweep of the cooperative step with the owner-side cache (dependent
minibatches, cache.cpp:137-208, run cooperatively): every rank walks a fixed
shuffled order of its own vertices in batches of b seeds; each step is the
captured peer-exchange step (cb_px_replay) followed by the owner-cached row
fetch (cb_px_gather_cached) with the shard in pinned host memory. Reports,
per kappa, the steady (second-epoch) miss rate, storage bytes per step (owner
cache misses x row bytes, the host link) and peer bytes per step (rows pulled
from other ranks' staging buffers). Run under torchrun (gloo; ranks may share
cuda:0 under MPS):
  torchrun --nproc-per-node 2 tools/px_kappa.py c3 [epochs] [batch] [requester_cache_rows]
With requester_cache_rows > 0 the rows other ranks own go through a second,
requester-side LRU and only its misses cross peer memory."""
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2310_12403_b200 as cb  # noqa: E402
from paper_2310_12403_b200.dist import PeerCoop, synth_shard  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
b = int(sys.argv[3]) if len(sys.argv) > 3 else cfg["batch"]
rcap = int(sys.argv[4]) if len(sys.argv) > 4 else 0
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
g = cb.Graph.generate_rmat(cfg["n"], cfg["m"], bench.GRAPH_SEED)
pm = cb.partition_random(g, world, bench.RUN_SEED)
mine = pm.members()[rank]
rng = np.random.default_rng(bench.RUN_SEED + rank)
order = mine[rng.permutation(len(mine))].astype(np.uint32)  # fixed training order
spe = max(1, len(order) // b)
steps = epochs * spe
cap = cfg["n"] // 10 // world  # |V|/10 rows of cache in total (acceptance.cpp:368)
L = len(cfg["fanouts"])
scfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, fanouts=cfg["fanouts"])
out = {"workload": cfg["workload"], "world": world, "batch_per_rank": b,
       "steps_per_epoch": spe, "epochs": epochs, "cache_rows_per_rank": cap,
       "requester_cache_rows_per_rank": rcap,
       "feature_tier": "shards in pinned host memory; cache rows in HBM", "sweep": []}
for kappa in (1, 4, 16, 64, 256, None):
    k = cb.KAPPA_INFINITY if kappa is None else kappa
    store = synth_shard(g, pm, rank, cfg["dim"], bench.FEAT_SEED, cfg["dtype"])
    pc = PeerCoop(g, pm, rank, L, scfg, max_seeds=b, store=store)
    store.set_tier(True)
    pc.enable_cache(cap, rcap)
    sched = cb.SeedSchedule.make(k, bench.RUN_SEED)
    pc.sample(order[:b], sched)
    pc.load_inputs()
    pc.finish()
    pc.capture(b, sched, rows=False)
    acc = {"acc": 0, "miss": 0, "peer_rows": 0, "rows": 0}
    lp = np.zeros(0, np.uint32)
    t0 = time.perf_counter()
    for step in range(steps):
        s0 = (step % spe) * b
        pc.step(order[s0:s0 + b], sched)
        owned, hits, misses = pc.load_inputs_cached(cb.hash_bits(step + 1, [rank]))
        if step >= spe:  # steady state: the second epoch on
            n_src, n_own = C.c_uint64(), C.c_uint64()
            pc.L.cb_px_sizes(pc._h, L - 1, C.byref(n_src), C.byref(n_own))
            if lp.size < n_src.value:
                lp = np.zeros(n_src.value, np.uint32)
            pc.L.cb_px_download(pc._h, L - 1, None, lp.ctypes.data_as(C.c_void_p), None, None)
            acc["acc"] += owned
            acc["miss"] += misses
            acc["rows"] += n_src.value
            if rcap:
                _, _, rmiss = pc.requester_stats()
                acc["peer_rows"] += rmiss  # only requester-cache misses cross
            else:
                acc["peer_rows"] += int(np.count_nonzero(lp[:n_src.value] != rank))
        sched = cb.schedule_advance(sched)
    pc.finish()
    dt = time.perf_counter() - t0
    t = torch.tensor([acc["acc"], acc["miss"], acc["peer_rows"], acc["rows"]],
                     dtype=torch.float64)
    dist.all_reduce(t)
    ms = torch.tensor([dt], dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    n_steady = max(1, steps - spe)
    rb = store.row_bytes
    out["sweep"].append({
        "kappa": "inf" if kappa is None else kappa,
        "steady_miss_rate": float(t[1] / max(t[0], 1)),
        "storage_bytes_per_step": float(t[1]) * rb / n_steady,
        "peer_bytes_per_step": float(t[2]) * rb / n_steady,
        "input_rows_per_seed": float(t[3]) / n_steady / (b * world),
        "wall_ms_per_step": 1e3 * float(ms) / steps})
    del pc, store
    dist.barrier()
if rank == 0:
    print(json.dumps(out))
dist.destroy_process_group()
