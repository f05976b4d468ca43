"""Shared harness for the multi-process cooperative tests (CPU gloo and GPU).

OracleEngine is the per-part compute stand-in for CPU runs: it evaluates one
block with the plain-C restatement and does bucketing / dedup / scatter in
numpy, so the tests exercise the product's DistCoop orchestration (count and
id all-to-allv, rank return, src_location assembly, feature fetch) over real
torch.distributed collectives without a GPU.
"""
import os
import socket
import traceback

import numpy as np
import torch
import torch.distributed as dist

from oracle import oracle as O


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleEngine:
    comm_device = torch.device("cpu")

    def __init__(self, g: O.CSR, owner: np.ndarray, world: int, kind: int, fanouts,
                 feat_seed: int, dim: int, dtype: str):
        self.g, self.owner, self.world = g, owner, world
        self.kind, self.fanouts = kind, list(fanouts)
        self.feat_seed, self.dim, self.dtype = feat_seed, dim, dtype
        self.row_bytes = dim * np.dtype(O.DTYPES[dtype][1]).itemsize
        self.blocks = {}

    def to_device(self, a):
        return torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32).copy())

    def to_host(self, t, n):
        return t[:n].numpy().view(np.uint32).copy()

    def empty_ids(self, n):
        return torch.empty(n, dtype=torch.int32)

    def sample_layer(self, l, D, n_d, schedule):
        d = self.to_host(D, n_d)
        s = O.Sched(schedule.kappa, schedule.z1, schedule.z2, schedule.iteration)
        b = O.sample_block(self.g, d, self.kind, self.fanouts[l], s, l)
        self.blocks[l] = b
        return self.to_device(b["src"]), len(b["src"])

    def bucket(self, src, n):
        s = self.to_host(src, n)
        own = self.owner[s]
        order = np.argsort(own, kind="stable")
        counts = np.bincount(own, minlength=self.world).tolist()
        return self.to_device(s[order]), torch.from_numpy(order.astype(np.int32)), counts

    def merge(self, l, recv, n):
        r = self.to_host(recv, n)
        uniq = np.unique(r)
        return self.to_device(uniq), len(uniq), self.to_device(np.searchsorted(uniq, r))

    def scatter(self, vals, perm, n):
        out = np.zeros(n, np.uint32)
        out[perm.numpy()] = self.to_host(vals, len(perm))
        return self.to_device(out)

    def block(self, l):
        return self.blocks[l]

    def gather_rows(self, ids, n):
        rows = O.feature_rows(self.feat_seed, self.dim, self.dtype, self.to_host(ids, n))
        return torch.from_numpy(rows.view(np.uint8).reshape(-1).copy())

    def scatter_rows(self, rows, perm, n, to_host=True):
        dt = O.DTYPES[self.dtype][1]
        r = rows.numpy().view(dt).reshape(-1, self.dim)
        out = np.zeros((n, self.dim), dt)
        out[perm.numpy()] = r
        return out


def check_rank(res, rows, exp, rank, world, L, feat_seed, dim, dtype):
    """Compare this rank's DistCoop result with the oracle coop_sample."""
    for l in range(L):
        for k in ("dst", "src", "edges", "dst_pos"):
            assert np.array_equal(res.blocks[l][k], exp["stacks"][rank][l][k]), (rank, l, k)
        ex, ref = res.exchanges[l], exp["exchanges"][l]
        assert list(ex.send_counts) == ref["send_counts"][rank].tolist(), (rank, l)
        assert ex.owner_row_count == int(ref["owner_row_counts"][rank])
        assert np.array_equal(ex.loc_part, ref["loc_part"][rank]), (rank, l)
        assert np.array_equal(ex.loc_row, ref["loc_row"][rank]), (rank, l)
    assert np.array_equal(res.owner_set, exp["owner_sets"][rank])
    want = O.feature_rows(feat_seed, dim, dtype, exp["stacks"][rank][L - 1]["src"])
    assert np.array_equal(rows.view(np.uint8), want.view(np.uint8)), rank


def run_worker(rank, world, port, fn, args, errq):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        fn(rank, world, *args)
        dist.barrier()
    except Exception:  # report to the parent, never hang the group
        errq.put(f"rank {rank}:\n{traceback.format_exc()}")
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def spawn(world, fn, args, timeout=300):
    ctx = torch.multiprocessing.get_context("spawn")
    errq = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=run_worker, args=(r, world, port, fn, args, errq))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout)
    for p in procs:
        if p.is_alive():
            p.kill()
            raise RuntimeError("distributed worker timed out")
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
