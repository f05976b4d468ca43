"""Debug: globaltimer stamps of one batch (CB_TRACE=1) of a bench config
(default c2; "flush" flushes L2 before the batch, "graph" replays the captured
batch). Prints per kernel the stamp offsets (us) relative to the first
stamp of the batch.  python tools/trace_batch.py [c4 [flush] [graph]]"""
import ctypes as C
import os
import sys

import numpy as np

os.environ["CB_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_12403_b200 as cb  # noqa: E402
from paper_2310_12403_b200 import _lib  # noqa: E402
from paper_2310_12403_b200.seeds import draw_from_pool  # noqa: E402
import bench  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
g = cb.Graph.generate_rmat(cfg["n"], cfg["m"], 42)
plan = cb.Plan(g, None, 3, cb.SamplerConfig(cb.SamplerKind.kLabor0, 10), 1024)
pool = np.arange(g.num_vertices, dtype=np.uint32)
s = cb.SeedSchedule.make(1, 1234)
flush = "flush" in sys.argv[2:]  # L2 flushed before the traced batch
graph = "graph" in sys.argv[2:]  # replays of the captured batch instead of eager launches
if graph:
    plan.capture([0, 1024], s, cb.MODE_INDEP)
for step in range(4):
    seeds = draw_from_pool(pool, 1024, 1234, cb.hash_bits(step, [0]))
    if flush and step == 3:
        import torch
        torch.empty(512 << 20, dtype=torch.uint8, device="cuda").zero_()
        torch.cuda.synchronize()
    if graph:
        plan.replay(seeds.ctypes.data, s, False, 1)
        plan.synchronize()
    else:
        plan.sample([seeds], s, cb.MODE_INDEP)
    s = cb.schedule_advance(s)
buf = np.zeros(32 * 64 * 8, np.uint64)
assert _lib.load().cb_plan_trace(plan._h, buf.ctypes.data_as(C.c_void_p), len(buf)) == 0
t = buf.reshape(32, 64, 8).astype(np.int64)
t0 = t[0, 0, 0]  # the batch's first stamp: frontier0, CTA 0 (older slots may hold stale stamps)
names = {0: "frontier0", 1: "mark0", 2: "post0", 3: "frontier1", 4: "mark1", 5: "post1",
         6: "frontier2", 7: "mark2", 8: "post2"}
# mark stamps: 0 start, 2 end of phase A (single-record tiles), 1 end; mark
# rows are every 16th CTA (row r = CTA 16 r)
for k, nm in names.items():
    # post: CTAs 0-31 = extract roles, 32-63 = emit roles
    for cta in ((list(range(0, 64, 1 if os.environ.get("TRACE_FIRST") else 4))
                 if nm.startswith("mark") else list(range(0, 64, 8)))
                if not nm.startswith("post") else
                [0, 1, 2, 8, 16, 31, 32, 33, 34, 40, 48, 63]):
        row = t[k, cta]
        if row[0] == 0:
            continue
        print(nm, cta, [round((x - t0) / 1000, 2) if x else None for x in row[:6 if nm.startswith("frontier") else 5]],
              # mark: phase-A tiles and prefilter survivors of the row's warp 0
              list(map(int, row[5:7])) if nm.startswith("mark") else "")
# latest end of any CTA per kernel (slot 63*8+7, atomicMax by every CTA)
print("kernel ends (us):", {nm: round((int(t[k, 63, 7]) - t0) / 1000, 2)
                             for k, nm in names.items() if t[k, 63, 7] > t0})
