"""GPU: cb_plan_result_async writes a batch's blocks and gathered rows into
pinned host memory in one kernel (csrc/result.cu); the parsed buffer must
equal the per-field downloads and the oracle, and a too-small buffer must
come back truncated with the size it needs."""
import numpy as np
import pytest

import paper_2310_12403_b200 as cb
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def osched(s):
    return O.Sched(s.kappa, s.z1, s.z2, s.iteration)


@pytest.fixture(scope="module")
def c1(gpu):
    n, m, seed = 1 << 16, 1 << 20, 42
    return cb.Graph.generate_rmat(n, m, seed), O.rmat(n, m, seed)


@pytest.mark.parametrize("kind,dtype,dim", [(cb.SamplerKind.kLabor0, "f16", 128),
                                            (cb.SamplerKind.kNs, "f32", 100),
                                            (cb.SamplerKind.kLabor0, "f32", 3)])
def test_result_buffer_matches_downloads(gpu, c1, kind, dtype, dim):
    import torch
    g, ref = c1
    store = cb.FeatureStore.synth(g, dim, 7, dtype)
    cfg = cb.SamplerConfig(kind, 10)
    rng = np.random.default_rng(dim)
    seeds = np.sort(rng.choice(ref.n, 700, replace=False)).astype(np.uint32)
    sched = cb.SeedSchedule.make(1, 5)
    plan = cb.Plan(g, None, 3, cfg, 1024)
    plan.sample([seeds], sched, cb.MODE_INDEP, sync=True)
    plan.capture(np.array([0, len(seeds)], np.uint64), sched, cb.MODE_INDEP, store)
    cap = 64 << 20
    buf = torch.empty(cap, dtype=torch.uint8).pin_memory()
    for step in range(3):
        sched = cb.schedule_advance(sched)
        s = np.sort(rng.choice(ref.n, len(seeds), replace=False)).astype(np.uint32)
        plan.replay(s.ctypes.data, sched, False, 3)
        plan.result_async(buf.data_ptr(), cap)
        plan.synchronize()
        res = cb.parse_result(buf.numpy(), np.float16 if dtype == "f16" else np.float32)
        # the copy-engine form: the same bytes (header + every section)
        buf2 = torch.zeros(cap, dtype=torch.uint8).pin_memory()
        if step != 1:
            plan.result_pack()  # else result_copy packs itself
        n = plan.result_copy(buf2.data_ptr(), cap)
        plan.synchronize()
        assert n == res["total_bytes"]
        a, b2 = buf.numpy()[:n], buf2.numpy()[:n]
        hdr = 8 * (5 + 3 * 3)
        assert np.array_equal(a[:hdr], b2[:hdr])
        res2 = cb.parse_result(buf2.numpy(), np.float16 if dtype == "f16" else np.float32)
        for l in range(3):
            for k in ("dst", "src", "edges", "dst_pos"):
                assert np.array_equal(res2["blocks"][l][k], res["blocks"][l][k])
        assert np.array_equal(res2["rows"].view(np.uint8), res["rows"].view(np.uint8))
        want = O.expand(ref, s, 3, int(kind), 10, osched(sched))
        for l in range(3):
            for k in ("dst", "src", "edges", "dst_pos"):
                assert np.array_equal(res["blocks"][l][k], want[l][k]), (step, l, k)
        exp = O.feature_rows(7, dim, dtype, want[2]["src"])
        assert np.array_equal(res["rows"].view(np.uint8).reshape(-1),
                              exp.view(np.uint8).reshape(-1))
        assert res["total_bytes"] <= plan.result_bytes(0, store.row_bytes)
    # truncation: header only, with the size needed
    small = torch.zeros(256, dtype=torch.uint8).pin_memory()
    plan.result_async(small.data_ptr(), 256)
    plan.synchronize()
    hd = small.numpy()[:40].view(np.uint64)
    assert int(hd[4]) == 1 and int(hd[3]) == res["total_bytes"]
    small.zero_()
    assert plan.result_copy(small.data_ptr(), 256) == res["total_bytes"]
    hd = small.numpy()[:40].view(np.uint64)
    assert int(hd[4]) == 1 and int(hd[3]) == res["total_bytes"]
    with pytest.raises(ValueError):
        cb.parse_result(small.numpy())
    # pageable memory is refused
    with pytest.raises(cb.InputError):
        plan.result_async(np.zeros(1024, np.uint8).ctypes.data, 1024)
