"""Per-phase device times of the eager peer-exchange step (dist.PeerCoop),
CUDA events on the plan stream between the C-ABI calls; run under torchrun
(gloo, ranks may share cuda:0 under MPS). Usage:
  torchrun --nproc-per-node N tools/px_diag.py c4 [steps]"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2310_12403_b200 as cb  # noqa: E402
from paper_2310_12403_b200.dist import PeerCoop, synth_shard  # noqa: E402
from paper_2310_12403_b200.seeds import draw_from_pool  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1]]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
g = cb.Graph.generate_rmat(cfg["n"], cfg["m"], bench.GRAPH_SEED)
pm = cb.partition_random(g, world, bench.RUN_SEED)
store = synth_shard(g, pm, rank, cfg["dim"], bench.FEAT_SEED, cfg["dtype"])
L = len(cfg["fanouts"])
pc = PeerCoop(g, pm, rank, L, cb.SamplerConfig(cb.SamplerKind.kLabor0, fanouts=cfg["fanouts"]),
              max_seeds=cfg["batch"], store=store)
mine = pm.members()[rank]
sched = cb.SeedSchedule.make(1, bench.RUN_SEED)
Lb = pc.L
times = {}
for s in range(steps):
    seeds = draw_from_pool(mine, cfg["batch"], bench.RUN_SEED, cb.hash_bits(s, [rank]))
    ev = []

    def mark(name):
        e = torch.cuda.Event(enable_timing=True)
        e.record(pc.stream)
        ev.append((name, e))
    sc = sched._c()
    mark("start")
    for l in range(L):
        Lb.cb_px_layer(pc._h, l, C.c_void_p(seeds.ctypes.data) if l == 0 else None,
                       len(seeds) if l == 0 else 0, C.byref(sc))
        mark(f"L{l}.sample+route")
        Lb.cb_px_barrier(pc._h)
        mark(f"L{l}.barrier1")
        Lb.cb_px_owner(pc._h, l)
        mark(f"L{l}.owner")
        Lb.cb_px_barrier(pc._h)
        mark(f"L{l}.barrier2")
        Lb.cb_px_locate(pc._h, l)
        mark(f"L{l}.locate")
    Lb.cb_px_gather(pc._h, store._h)
    mark("gather")
    pc.finish()
    if s >= 2:
        for (a, ea), (b, eb) in zip(ev, ev[1:]):
            times.setdefault(b, []).append(ea.elapsed_time(eb) * 1e3)
    sched = cb.schedule_advance(sched)
out = {k: round(float(np.median(v)), 1) for k, v in times.items()}
print(json.dumps({"rank": rank, "world": world, "us": out, "total": round(sum(out.values()), 1)}))
dist.destroy_process_group()
