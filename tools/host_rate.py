"""Is the in-flight bench host-bound? Times the host issue loop of K graph
replays over S plans (c2) against the device time of the same K steps."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2310_12403_b200 as cb  # noqa: E402
from paper_2310_12403_b200.seeds import draw_from_pool  # noqa: E402

c = bench.CONFIGS["c2"]
g = cb.Graph.generate_rmat(c["n"], c["m"], bench.GRAPH_SEED)
store = cb.FeatureStore.synth(g, c["dim"], 5)
scfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, fanouts=c["fanouts"])
b, L, K, S = 1024, 3, 400, 8
pool = np.arange(g.num_vertices, dtype=np.uint32)
seeds = np.stack([draw_from_pool(pool, b, 1, i) for i in range(K)])
d = torch.from_numpy(seeds.view(np.int32)).cuda()
off = np.array([0, b], np.uint64)
sched = cb.SeedSchedule.make(1, 1)
plans = []
for _ in range(S):
    p = cb.Plan(g, None, L, scfg, b)
    p.sample([seeds[0]], sched, cb.MODE_INDEP)
    p.capture(off, sched, cb.MODE_INDEP, store)
    plans.append(p)
scheds = [sched]
for i in range(K):
    scheds.append(cb.schedule_advance(scheds[-1]))
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(K):
        plans[i % S].replay(d.data_ptr() + i * b * 4, scheds[i], True, 3)
    t1 = time.perf_counter()
    for p in plans:
        p.synchronize()
    t2 = time.perf_counter()
    print(f"issue {1e6 * (t1 - t0) / K:.1f} us/step, total {1e6 * (t2 - t0) / K:.1f} us/step")
