"""Experiment: throughput of S independent minibatches in flight (S plans,
S streams, CUDA-graph replays), c2, no per-step L2 flush."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_12403_b200 as cb  # noqa: E402
from paper_2310_12403_b200.seeds import draw_from_pool  # noqa: E402

n, m, b, K = 2449029, 61859140, 1024, 64
g = cb.Graph.generate_rmat(n, m, 42)
store = cb.FeatureStore.synth(g, 100, 7, "f32")
cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, fanouts=[10, 10, 10])
pool = np.arange(n, dtype=np.uint32)
seeds = np.stack([draw_from_pool(pool, b, 1234, cb.hash_bits(s, [0])) for s in range(K)])
d = torch.from_numpy(seeds.view(np.int32)).cuda()
sch = [cb.SeedSchedule.make(1, 1234)]
for _ in range(K):
    sch.append(cb.schedule_advance(sch[-1]))
for S in (1, 2, 4, 6, 8, 12):
    plans = []
    for s in range(S):
        p = cb.Plan(g, None, 3, cfg, b)
        p.sample([seeds[0]], sch[0], cb.MODE_INDEP, sync=True)
        p.capture(np.array([0, b], np.uint64), sch[0], cb.MODE_INDEP, store)
        plans.append(p)
    streams = [torch.cuda.ExternalStream(p.stream) for p in plans]
    for it in range(2):
        torch.cuda.synchronize()
        master = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(master)
        for st in streams:
            st.wait_event(e0)
        for i in range(K):
            plans[i % S].replay(d.data_ptr() + i * b * 4, sch[i], True, 3)
        for st in streams:
            ev = torch.cuda.Event()
            ev.record(st)
            master.wait_event(ev)
        e1.record(master)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    print(f"S={S}: {1e3 * ms / K:.1f} us/step  {K * b / (ms / 1e3) / 1e6:.2f} M seeds/s", flush=True)
    del plans, streams
