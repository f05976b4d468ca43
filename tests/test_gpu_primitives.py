"""GPU: the multi-process exchange primitives against numpy restatements of
build_exchange's routing (coop.cpp:35-62): stable bucketing by owner, owner
side sort+unique with ranks, scatter."""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_2310_12403_b200 as cb
from paper_2310_12403_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def plan(gpu):
    g = cb.Graph.generate_rmat(1 << 16, 1 << 18, 3)
    h = C.c_void_p()
    fo = np.array([10, 10], np.uint32)
    assert gpu.cb_plan_create_dist(g._h, 4, 2, 2, fo.ctypes.data_as(C.c_void_p), 1 << 16,
                                   C.byref(h)) == 0, gpu.cb_last_error()
    yield g, h
    gpu.cb_plan_destroy(h)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


@pytest.mark.parametrize("P", [1, 2, 3, 5, 8, 64])
@pytest.mark.parametrize("n", [0, 1, 100, 4096, 4097, 50000])
def test_bucket_by_owner(plan, P, n):
    g, h = plan
    L = _lib.load()
    rng = np.random.default_rng(P * 1000 + n)
    ids = np.sort(rng.choice(1 << 16, size=n, replace=False)).astype(np.uint32)
    owner = rng.integers(0, P, 1 << 16).astype(np.uint32)
    d_ids, d_own = dev(ids), dev(owner)
    out = torch.zeros(max(n, 1), dtype=torch.int32, device="cuda")
    perm = torch.zeros(max(n, 1), dtype=torch.int32, device="cuda")
    counts = np.zeros(P, np.uint64)
    rc = L.cb_bucket_by_owner(h, C.c_void_p(d_ids.data_ptr()), n, C.c_void_p(d_own.data_ptr()),
                              P, C.c_void_p(out.data_ptr()), C.c_void_p(perm.data_ptr()),
                              counts.ctypes.data_as(C.c_void_p))
    assert rc == 0, L.cb_last_error()
    order = np.argsort(owner[ids], kind="stable")
    assert np.array_equal(counts, np.bincount(owner[ids], minlength=P).astype(np.uint64))
    assert np.array_equal(out[:n].cpu().numpy().view(np.uint32), ids[order])
    assert np.array_equal(perm[:n].cpu().numpy(), order.astype(np.int32))


@pytest.mark.parametrize("n", [0, 1, 1000, 70000])
def test_merge_owned_and_scatter(plan, n):
    g, h = plan
    L = _lib.load()
    rng = np.random.default_rng(n)
    recv = rng.integers(0, 1 << 16, n).astype(np.uint32)
    d_recv = dev(recv)
    nxt = torch.zeros(max(n, 1), dtype=torch.int32, device="cuda")
    rank = torch.zeros(max(n, 1), dtype=torch.int32, device="cuda")
    n_next = C.c_uint64()
    for layer in (0, 1):  # repeated use must leave the bitmap clean
        rc = L.cb_merge_owned(h, layer, C.c_void_p(d_recv.data_ptr()), n,
                              C.c_void_p(nxt.data_ptr()), max(n, 1), C.byref(n_next),
                              C.c_void_p(rank.data_ptr()))
        assert rc == 0, L.cb_last_error()
        uniq = np.unique(recv)
        assert n_next.value == len(uniq)
        assert np.array_equal(nxt[:len(uniq)].cpu().numpy().view(np.uint32), uniq)
        assert np.array_equal(rank[:n].cpu().numpy(), np.searchsorted(uniq, recv).astype(np.int32))
    perm = rng.permutation(n).astype(np.int32)
    out = torch.zeros(max(n, 1), dtype=torch.int32, device="cuda")
    d_perm = dev(perm)
    assert L.cb_scatter_u32(h, C.c_void_p(d_recv.data_ptr()), C.c_void_p(d_perm.data_ptr()), n,
                            C.c_void_p(out.data_ptr())) == 0
    want = np.zeros(n, np.uint32)
    want[perm] = recv
    assert np.array_equal(out[:n].cpu().numpy().view(np.uint32), want)
