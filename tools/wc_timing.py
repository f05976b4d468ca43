"""Timing breakdown of GPU work_curve pieces (tools; not a test)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2310_12403_b200 as cb  # noqa: E402
from paper_2310_12403_b200 import analysis as A  # noqa: E402

c = bench.CONFIGS["c1"]
g = cb.Graph.generate_rmat(c["n"], c["m"], bench.GRAPH_SEED)
sizes = [64 << i for i in range(8)]
cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0)
for P, b in ((1, 8192), (16, 8192), (16, 512), (1, 512)):
    pl = cb.Plan(g, None, 3, cfg, b, parts=P)
    seeds = [A.draw_seeds(g.num_vertices, b, 49, t) for t in range(P)]
    sc = [cb.SeedSchedule.plain(t) for t in range(P)]
    pl.sample_multi(seeds, sc)
    t0 = time.time()
    for i in range(10):
        pl.sample_multi(seeds, sc)
    dt = (time.time() - t0) / 10
    prof = pl.profile(seeds, sc[0], cb.MODE_INDEP)
    print(f"P={P} b={b}: sample_multi {dt * 1e3:.2f} ms; kernels sum {sum(prof):.3f} ms "
          f"n={len(prof)} top={sorted(prof)[-4:]}")
    print("  per-launch:", [round(x, 3) for x in prof[:14]])
for per in (8, 16, 50):
    t0 = time.time()
    A.work_curve(g, cfg, sizes, 50, 3, 49, trials_per_launch=per)
    print("curve", per, time.time() - t0)
