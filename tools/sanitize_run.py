"""Small end-to-end workload for compute-sanitizer (tests/test_gpu_sanitizer.py):
every kernel family once on small inputs — R-MAT generation, partition,
LABOR/NS/FULL/RW expand (plain + smoothed), coop P=3 with gather, CUDA-graph
replay, LRU cache with rows, the training step."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_12403_b200 as cb  # noqa: E402

n, m = 3000, 24000
g = cb.Graph.generate_rmat(n, m, 5)
rng = np.random.default_rng(0)
seeds = np.sort(rng.choice(n, 200, replace=False)).astype(np.uint32)
for kind in (cb.SamplerKind.kFull, cb.SamplerKind.kNs, cb.SamplerKind.kLabor0, cb.SamplerKind.kRw):
    for kappa in (1, 4):
        sched = cb.schedule_advance(cb.SeedSchedule.make(kappa, 3))
        cb.expand(g, seeds, 2, cb.SamplerConfig(kind, 4), sched)
pm = cb.partition_random(g, 3, 2)
store = cb.FeatureStore.synth(g, 12, 1, "f32", pm)
per = [seeds[pm.owner[seeds] == p] for p in range(3)]
cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, 5)
cb.load_inputs(g, pm, per, 3, cfg, cb.SeedSchedule.plain(2), store)
plan = cb.Plan(g, None, 3, cfg, 200)
s0 = cb.SeedSchedule.plain(1)
plan.sample([seeds], s0, cb.MODE_INDEP)
st1 = cb.FeatureStore.synth(g, 12, 1, "f32")
plan.capture(np.array([0, 200], np.uint64), s0, cb.MODE_INDEP, st1)
import torch  # noqa: E402
d = torch.from_numpy(seeds.view(np.int32)).cuda()
for i in range(2):
    plan.replay(d.data_ptr(), s0, True, 3)
plan.synchronize()
cache = cb.LruCache(300, n, 0, 48)
cache.access_plan(plan, 0, 77, store=st1)
cache.access_trace(rng.integers(0, n, 2000).astype(np.uint32))
f64 = cb.FeatureStore.synth(g, 6, 1, "f64", pm)
model = cb.GcnModel.init(6, 5, 4, 2, 2)
cb.coop_train_step(g, pm, per, 2, cfg, cb.SeedSchedule.plain(3), model, f64, 4)
# labor_mark phase A (single-record hub tiles by bulk copy) and phase B: a
# hub with 6000 in-neighbours among ordinary vertices
nh = 8000
src = [np.arange(1, 6001, dtype=np.uint32)]
dst = [np.zeros(6000, np.uint32)]
src.append(rng.integers(0, nh, 40000).astype(np.uint32))
dst.append(rng.integers(1, nh, 40000).astype(np.uint32))
s_all, d_all = np.concatenate(src), np.concatenate(dst)
order = np.lexsort((s_all, d_all))
s_all, d_all = s_all[order], d_all[order]
indptr = np.zeros(nh + 1, np.uint64)
np.add.at(indptr, d_all.astype(np.int64) + 1, 1)
indptr = np.cumsum(indptr).astype(np.uint64)
gh = cb.Graph.from_csr(indptr, s_all)
hseeds = np.concatenate([[0], rng.choice(np.arange(1, nh), 300, replace=False)]).astype(np.uint32)
hp = cb.Plan(gh, None, 3, cb.SamplerConfig(cb.SamplerKind.kLabor0, 10), len(hseeds))
hp.sample([hseeds], cb.SeedSchedule.plain(5), cb.MODE_INDEP)
# the batch result by the result kernel and by pack + copy-engine copy
hs = cb.FeatureStore.synth(gh, 8, 1, "f16")
hp.gather(hs)
pin = torch.empty(8 << 20, dtype=torch.uint8).pin_memory()
hp.result_async(pin.data_ptr(), pin.numel())
hp.result_pack()
hp.result_copy(pin.data_ptr(), pin.numel())
hp.synchronize()
# smoothed decisions in a forced guard band, resolved on the host (re-samples)
hp.set_guard(1e-2, perturb=True)
hp.sample([hseeds], cb.schedule_advance(cb.SeedSchedule.make(4, 9)), cb.MODE_INDEP)
print("sanitize workload done")
