"""Multi-process cooperative minibatching: one process per GPU, one part per
rank (Alg. 1; coop.cpp:68-106 with the in-memory exchange of
build_exchange, coop.cpp:25-64, replaced by all-to-allv between ranks).

Per layer l on rank p:
  1. engine.sample_layer(l, D_p)   -> sorted unique src list S~_p (device)
  2. engine.bucket(S~_p)           -> ids bucketed by owner, perm, counts
  3. all_to_all(counts); all_to_all(ids)        [torch.distributed: NCCL]
  4. engine.merge(l, received)     -> D_p^{l+1} (sorted unique) + row of
                                      every received id in it
  5. all_to_all(rows back)         -> src_location[p][j] = (owner, row)
Feature loading (coop.cpp:457-467): the owner gathers the rows requested by
the last layer's ids from its shard and returns them in request order; the
requester scatters them to src order (all_to_all_forward).

The engine does the per-part compute. ``CudaEngine`` runs the sm_100a
kernels through the C-ABI; the CPU tests run the same orchestration with an
oracle-backed engine over the gloo backend.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .coopbatch import (FeatureStore, Graph, PartitionMap, SamplerConfig, SeedSchedule,
                        _check, _DT)


@dataclass
class DistExchange:
    """This rank's row of an ExchangeRecord (coop.hpp:25-37)."""
    layer: int
    send_counts: list[int]         # send_counts[p][*] for this rank p
    owner_row_count: int           # owner_row_counts[p]
    loc_part: np.ndarray           # src_location[p][*].part
    loc_row: np.ndarray            # src_location[p][*].row


@dataclass
class DistSample:
    blocks: list[dict] = field(default_factory=list)
    exchanges: list[DistExchange] = field(default_factory=list)
    owner_set: np.ndarray | None = None


def _i32(t: torch.Tensor) -> torch.Tensor:
    return t.view(torch.int32) if t.dtype != torch.int32 else t


class DistCoop:
    def __init__(self, engine, group=None):
        self.e = engine
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._last = None

    def _a2a(self, out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits):
        dist.all_to_all_single(out, inp, output_split_sizes=list(out_splits),
                               input_split_sizes=list(in_splits), group=self.group)

    def _exchange_counts(self, counts) -> list[int]:
        send = torch.tensor(counts, dtype=torch.int64, device=self.e.comm_device)
        recv = torch.empty(self.world, dtype=torch.int64, device=self.e.comm_device)
        dist.all_to_all_single(recv, send, group=self.group)
        return recv.tolist()

    def sample(self, seeds, num_layers: int, schedule: SeedSchedule,
               keep_blocks: bool = True, records: bool = True) -> DistSample:
        """One cooperative step. `seeds` is a host array or a device tensor
        (int32 view of u32 ids). records=False keeps the exchange on the
        device only (no host ExchangeRecord / owner set), for timing."""
        out = DistSample()
        if isinstance(seeds, torch.Tensor):
            D, n_d = seeds, seeds.numel()
        else:
            D = self.e.to_device(np.ascontiguousarray(seeds, dtype=np.uint32))
            n_d = len(seeds)
        for l in range(num_layers):
            src, n_src = self.e.sample_layer(l, D, n_d, schedule)
            bucketed, perm, counts = self.e.bucket(src, n_src)
            rcounts = self._exchange_counts(counts)
            recv = self.e.empty_ids(sum(rcounts))
            self._a2a(_i32(recv), _i32(bucketed), rcounts, counts)
            D, n_d, ranks = self.e.merge(l, recv, sum(rcounts))
            back = self.e.empty_ids(sum(counts))
            self._a2a(_i32(back), _i32(ranks), counts, rcounts)
            loc_row = self.e.scatter(back, perm, n_src)
            if records:
                part = np.repeat(np.arange(self.world, dtype=np.uint32), counts)
                loc_part = np.zeros(n_src, np.uint32)
                loc_part[self.e.to_host(perm, n_src)] = part
                out.exchanges.append(DistExchange(
                    l, counts, n_d, loc_part, self.e.to_host(loc_row, n_src).astype(np.uint64)))
            if keep_blocks:
                out.blocks.append(self.e.block(l))
            self._last = (recv, sum(rcounts), rcounts, perm, counts, n_src)
        self.n_owned = n_d
        if records:
            out.owner_set = self.e.to_host(D, n_d)
        return out

    def load_inputs(self, to_host: bool = True):
        """Rows of this rank's input vertices (src of the last block), in src
        order: owner-side gather of the requested ids, all-to-allv back,
        requester-side scatter (all_to_all_forward, coop.cpp:145-159).
        to_host=False returns the device tensor (bytes) instead."""
        recv, n_recv, rcounts, perm, counts, n_src = self._last
        rb = self.e.row_bytes
        rows = self.e.gather_rows(recv, n_recv)              # owner side, request order
        back = torch.empty(sum(counts) * rb, dtype=torch.uint8, device=self.e.comm_device)
        self._a2a(back, rows, [c * rb for c in counts], [c * rb for c in rcounts])
        return self.e.scatter_rows(back, perm, n_src, to_host=to_host)


class CudaEngine:
    """Per-part compute through libcoopbatch_b200 (sm_100a kernels)."""

    def __init__(self, g: Graph, pm: PartitionMap, rank: int, num_layers: int,
                 cfg: SamplerConfig, max_seeds: int, store: FeatureStore | None = None,
                 comm_device: str | None = None):
        self.L = _lib.load()
        self.g, self.rank, self.world = g, rank, pm.num_parts
        self.device = torch.device(f"cuda:{g.device}")
        # ids/rows cross ranks on this device (NCCL); "cpu" stages them for gloo
        self.comm_device = torch.device(comm_device) if comm_device else self.device
        fo = np.asarray(cfg.layer_fanouts(num_layers), dtype=np.uint32)
        h = C.c_void_p()
        _check(self.L.cb_plan_create_dist(g._h, pm.num_parts, num_layers, int(cfg.kind),
                                          fo.ctypes.data_as(C.c_void_p), max_seeds,
                                          C.byref(h)))
        self._h = h
        self.owner = torch.from_numpy(pm.owner.view(np.int32)).to(self.device)
        self.store = store
        self.row_bytes = store.row_bytes if store is not None else 0

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                self.L.cb_plan_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown: the loader may be gone
            pass

    # -- helpers --------------------------------------------------------------
    def _dev(self, t: torch.Tensor) -> torch.Tensor:
        """Device copy of a torch tensor, complete before the library's own
        (non-blocking) plan stream reads it."""
        t = t if t.device == self.device else t.to(self.device)
        torch.cuda.current_stream(self.device).synchronize()
        return t

    def _comm(self, t: torch.Tensor) -> torch.Tensor:
        return t if t.device == self.comm_device else t.to(self.comm_device)

    def to_device(self, a: np.ndarray) -> torch.Tensor:
        return torch.from_numpy(a.view(np.int32)).to(self.device)

    def to_host(self, t: torch.Tensor, n: int) -> np.ndarray:
        return t[:n].cpu().numpy().view(np.uint32).copy()

    def empty_ids(self, n: int) -> torch.Tensor:
        return torch.empty(max(n, 1), dtype=torch.int32, device=self.comm_device)[:n]

    # -- engine interface -----------------------------------------------------
    def sample_layer(self, l, D, n_d, schedule: SeedSchedule):
        D = self._dev(D)  # also orders torch-side writes before the plan stream
        n_src = C.c_uint64()
        s = schedule._c()
        _check(self.L.cb_plan_sample_layer(self._h, l, C.c_void_p(D.data_ptr()), n_d,
                                           C.byref(s), C.byref(n_src)))
        ptr = C.c_void_p()
        _check(self.L.cb_plan_layer_src(self._h, l, C.byref(ptr)))
        src = torch.empty(max(n_src.value, 1), dtype=torch.int32, device=self.device)
        _check(self.L.cb_memcpy(C.c_void_p(src.data_ptr()), ptr, n_src.value * 4,
                                self.g.device))
        return src[: n_src.value], n_src.value

    def bucket(self, src, n):
        torch.cuda.current_stream(self.device).synchronize()
        out = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        perm = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        counts = np.zeros(self.world, np.uint64)
        _check(self.L.cb_bucket_by_owner(self._h, C.c_void_p(src.data_ptr()), n,
                                         C.c_void_p(self.owner.data_ptr()), self.world,
                                         C.c_void_p(out.data_ptr()),
                                         C.c_void_p(perm.data_ptr()),
                                         counts.ctypes.data_as(C.c_void_p)))
        return self._comm(out[:n]), perm[:n], [int(c) for c in counts]

    def merge(self, l, recv, n_recv):
        recv = self._dev(recv)
        nxt = torch.empty(max(n_recv, 1), dtype=torch.int32, device=self.device)
        rank = torch.empty(max(n_recv, 1), dtype=torch.int32, device=self.device)
        n_next = C.c_uint64()
        _check(self.L.cb_merge_owned(self._h, l, C.c_void_p(recv.data_ptr()), n_recv,
                                     C.c_void_p(nxt.data_ptr()), max(n_recv, 1),
                                     C.byref(n_next), C.c_void_p(rank.data_ptr())))
        return nxt[: n_next.value], n_next.value, self._comm(rank[:n_recv])

    def scatter(self, vals, perm, n):
        vals = self._dev(vals)
        out = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        _check(self.L.cb_scatter_u32(self._h, C.c_void_p(vals.data_ptr()),
                                     C.c_void_p(perm.data_ptr()), n,
                                     C.c_void_p(out.data_ptr())))
        return out[:n]

    def block(self, l) -> dict:
        sz = np.zeros(6, np.uint64)
        _check(self.L.cb_layer_sizes(self._h, 0, l, sz.ctypes.data_as(C.c_void_p)))
        nd, ns, ne = int(sz[0]), int(sz[1]), int(sz[2])
        dst, src = np.zeros(nd, np.uint32), np.zeros(ns, np.uint32)
        edges, dpos = np.zeros((ne, 2), np.uint32), np.zeros(nd, np.uint32)
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        _check(self.L.cb_download_block(self._h, 0, l, p(dst), p(src), p(edges), p(dpos)))
        return {"layer": l, "dst": dst, "src": src, "edges": edges, "dst_pos": dpos}

    def gather_rows(self, ids, n):
        ids = self._dev(ids)
        out = torch.empty(max(n, 1) * self.row_bytes, dtype=torch.uint8, device=self.device)
        _check(self.L.cb_gather_rows(self.store._h, C.c_void_p(ids.data_ptr()), n,
                                     C.c_void_p(out.data_ptr()), None))
        return self._comm(out[: n * self.row_bytes])

    def scatter_rows(self, rows, perm, n, to_host: bool = True):
        rows = self._dev(rows)
        out = torch.empty(max(n, 1) * self.row_bytes, dtype=torch.uint8, device=self.device)
        _check(self.L.cb_scatter_rows(self._h, C.c_void_p(rows.data_ptr()),
                                      C.c_void_p(perm.data_ptr()), n, self.row_bytes,
                                      C.c_void_p(out.data_ptr())))
        if not to_host:
            return out[: n * self.row_bytes]
        dt = _DT[self.store.dtype][1]
        return out[: n * self.row_bytes].cpu().numpy().view(dt).reshape(n, self.store.dim)


def synth_shard(g: Graph, pm: PartitionMap, part: int, dim: int, seed: int,
                dtype: str = "f32") -> FeatureStore:
    """Feature rows of one part only (FeatureStore::synth restricted to the
    part's members, coop.cpp:359-376)."""
    h = C.c_void_p()
    _check(_lib.load().cb_features_synth_shard(g._h, pm._h, part, dim, _DT[dtype][0], seed,
                                               C.byref(h)))
    return FeatureStore(g, h, dim, dtype, pm)


class PeerCoop:
    """One part per rank with the exchange done in peer memory (cb_px_*,
    csrc/exchange.cu): each rank's src ids are OR-ed straight into their
    owners' exchange bitmaps over NVLink (CUDA IPC mappings), owners extract
    their sorted sets in place, requesters read their ranks back from the
    owners' bitmaps, and input rows are pulled from the owners' shards
    requester-aligned. No counts cross ranks and the host never waits: the
    only cross-rank operation is a barrier between the three phases of a
    layer. `barrier="device"` (default) is cb_px_barrier, a one-warp kernel
    on flags in the IPC region, so a whole step can be captured as one CUDA
    graph per rank (`capture` / `step`); "nccl" is an NCCL all-reduce of one
    element on the plan stream, "host" a stream sync plus a process-group
    barrier."""

    HANDLE = 64

    def __init__(self, g: Graph, pm: PartitionMap, rank: int, num_layers: int,
                 cfg: SamplerConfig, max_seeds: int, store: FeatureStore | None = None,
                 group=None, barrier: str = "device", direct_rows: bool = False):
        if barrier not in ("device", "nccl", "host"):
            raise ValueError("PeerCoop: barrier must be 'device', 'nccl' or 'host'")
        self.L = _lib.load()
        self.g, self.pm, self.rank, self.group = g, pm, rank, group
        self.world = dist.get_world_size(group)
        if pm.num_parts != self.world:
            raise ValueError("PeerCoop: partition part count must equal the world size")
        self.num_layers, self.store = num_layers, store
        self.device = torch.device(f"cuda:{g.device}")
        fo = np.asarray(cfg.layer_fanouts(num_layers), dtype=np.uint32)
        h = C.c_void_p()
        _check(self.L.cb_plan_create_dist(g._h, self.world, num_layers, int(cfg.kind),
                                          fo.ctypes.data_as(C.c_void_p), max_seeds,
                                          C.byref(h)))
        self._h = h
        buf = (C.c_ubyte * self.HANDLE)()
        _check(self.L.cb_px_setup(h, pm._h, rank, buf))
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(buf), group=group)
        for q in range(self.world):
            if q != rank:
                hq = (C.c_ubyte * self.HANDLE).from_buffer_copy(handles[q])
                _check(self.L.cb_px_connect(h, q, hq))
        if store is not None and direct_rows:
            # rows read in place from the peers' shards (one mapping of a
            # shard per process: a second PeerCoop over the same store
            # cannot map it again)
            fb, r0 = (C.c_ubyte * self.HANDLE)(), C.c_uint64()
            _check(self.L.cb_features_export(store._h, fb, C.byref(r0)))
            fh = [None] * self.world
            dist.all_gather_object(fh, (bytes(fb), r0.value), group=group)
            for q in range(self.world):
                hq = (C.c_ubyte * self.HANDLE).from_buffer_copy(fh[q][0])
                _check(self.L.cb_px_connect_features(h, q, hq, fh[q][1], store._h))
        elif store is not None:
            # owner staging: owners load their requested rows, requesters pull
            sb = (C.c_ubyte * self.HANDLE)()
            _check(self.L.cb_px_setup_staging(h, store._h, sb))
            sh = [None] * self.world
            dist.all_gather_object(sh, bytes(sb), group=group)
            for q in range(self.world):
                if q != rank:
                    hq = (C.c_ubyte * self.HANDLE).from_buffer_copy(sh[q])
                    _check(self.L.cb_px_connect_staging(h, q, hq))
        self.stream = torch.cuda.ExternalStream(self.L.cb_plan_stream(h), device=self.device)
        self._nccl = dist.get_backend(group) == "nccl"
        if barrier == "nccl" and not self._nccl:
            raise ValueError("PeerCoop: barrier='nccl' needs an NCCL process group")
        self._barrier = barrier
        self._captured = False
        self._tok = torch.zeros(1, device=self.device if self._nccl else "cpu")
        dist.barrier(group=group)  # every mapping is open before anyone writes

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                self.L.cb_plan_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown: the loader may be gone
            pass

    def barrier(self):
        if self._barrier == "device":
            _check(self.L.cb_px_barrier(self._h))
        elif self._barrier == "nccl":
            with torch.cuda.stream(self.stream):
                dist.all_reduce(self._tok, group=self.group)
        else:
            _check(self.L.cb_synchronize(self._h))
            dist.barrier(group=self.group)

    def sample(self, seeds, schedule: SeedSchedule):
        """One cooperative step for this rank's seeds (host u32 array or a
        device tensor), all phases stream-ordered on the plan stream."""
        if isinstance(seeds, torch.Tensor):
            ptr, n = seeds.data_ptr(), seeds.numel()
            # the plan stream copies the seeds: order it after their producer
            self.stream.wait_stream(torch.cuda.current_stream(self.device))
            self._seeds = seeds  # keep alive until the copy is enqueued
        else:
            self._seeds = np.ascontiguousarray(seeds, dtype=np.uint32)
            ptr, n = self._seeds.ctypes.data, len(self._seeds)
        s = schedule._c()
        for l in range(self.num_layers):
            _check(self.L.cb_px_layer(self._h, l, C.c_void_p(ptr) if l == 0 else None,
                                      n if l == 0 else 0, C.byref(s)))
            self.barrier()
            _check(self.L.cb_px_owner(self._h, l))
            self.barrier()
            _check(self.L.cb_px_locate(self._h, l))

    def capture(self, n_seeds: int, schedule: SeedSchedule, rows: bool = True):
        """Capture the whole step (L layers with their device barriers, plus
        the row pull when `rows` and a store is set) as one CUDA graph per
        rank (cb_px_capture). Needs barrier="device" and one eager step
        (`sample`) on every rank first; every rank captures together."""
        if self._barrier != "device":
            raise ValueError("PeerCoop.capture needs barrier='device'")
        store = self.store._h if (rows and self.store is not None) else None
        _check(self.L.cb_px_finish(self._h))
        dist.barrier(group=self.group)  # no peer writes into our slots while they are reset
        _check(self.L.cb_px_capture(self._h, n_seeds, C.byref(schedule._c()), store))
        dist.barrier(group=self.group)
        self._captured = True

    def step(self, seeds, schedule: SeedSchedule):
        """One captured step (cb_px_replay): seeds (host u32 array of the
        captured length, or a device tensor) and variates copied on the plan
        stream, then one graph launch; nothing waits on the host."""
        if not self._captured:
            raise RuntimeError("PeerCoop.step: call capture() first")
        if isinstance(seeds, torch.Tensor):
            self.stream.wait_stream(torch.cuda.current_stream(self.device))
            self._seeds = seeds
            ptr, on_dev = seeds.data_ptr(), 1
        else:
            self._seeds = np.ascontiguousarray(seeds, dtype=np.uint32)
            ptr, on_dev = self._seeds.ctypes.data, 0
        _check(self.L.cb_px_replay(self._h, C.c_void_p(ptr), on_dev, C.byref(schedule._c())))

    def enable_cache(self, capacity: int, requester_capacity: int = 0):
        """Owner-side LRU cache of `capacity` rows (HBM) in front of this rank's
        shard (cb_px_set_cache) and, with requester_capacity > 0, a
        requester-side LRU for the rows other ranks own (only its misses cross
        NVLink; cb_px_set_requester_cache): see load_inputs_cached."""
        from .cache import LruCache
        if self.store is None:
            raise ValueError("PeerCoop.enable_cache needs the rank's feature shard")
        self.cache = LruCache(capacity, self.g.num_vertices, self.g.device,
                              row_bytes=self.store.row_bytes)
        _check(self.L.cb_px_set_cache(self._h, self.cache._h))
        self.rcache = None
        if requester_capacity > 0:
            self.rcache = LruCache(requester_capacity, self.g.num_vertices, self.g.device,
                                   row_bytes=self.store.row_bytes)
            _check(self.L.cb_px_set_requester_cache(self._h, self.rcache._h))

    def enable_clock_cache(self, capacity: int, ways: int = 8):
        """The CLOCK cache (cb_ccache_*) in front of this owner's staging: the
        cached fetch becomes part of the captured step (no host round trip).
        Call before capture()."""
        from .cache import ClockCache
        if self.store is None:
            raise ValueError("PeerCoop.enable_clock_cache needs the rank's feature shard")
        self.ccache = ClockCache(capacity, self.store.row_bytes, self.g.device, ways)
        _check(self.L.cb_px_set_clock_cache(self._h, self.ccache._h))
        self._captured = False

    def requester_stats(self) -> tuple[int, int, int]:
        """Last cached fetch, requester side: (remote rows, hits, misses)."""
        r, h, m = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(self.L.cb_px_requester_stats(self._h, C.byref(r), C.byref(h), C.byref(m)))
        return r.value, h.value, m.value

    def load_inputs_cached(self, order_key: int) -> tuple[int, int, int]:
        """The owner-side cached fetch of this step (cb_px_gather_cached): this
        owner's set S^L_q goes through its LRU in access_order(S^L_q, order_key)
        (misses from the shard, HBM or host tier), then every rank pulls its
        rows from the owners' staged rows. Returns (owned rows, hits, misses)
        of this owner."""
        o, h, m = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(self.L.cb_px_gather_cached(self._h, order_key, C.byref(o), C.byref(h),
                                          C.byref(m)))
        return o.value, h.value, m.value

    def load_inputs(self):
        """all_to_all_forward: rows of the input vertices pulled from the
        owners' shards into the plan's row buffer (shards are static, so no
        barrier is needed)."""
        _check(self.L.cb_px_gather(self._h, self.store._h))

    def finish(self):
        _check(self.L.cb_px_finish(self._h))

    # -- results (host) --------------------------------------------------------
    def result(self) -> DistSample:
        self.finish()
        out = DistSample()
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        for l in range(self.num_layers):
            sz = np.zeros(6, np.uint64)
            _check(self.L.cb_layer_sizes(self._h, 0, l, p(sz)))
            nd, ns, ne = int(sz[0]), int(sz[1]), int(sz[2])
            dst, src = np.zeros(nd, np.uint32), np.zeros(ns, np.uint32)
            edges, dpos = np.zeros((ne, 2), np.uint32), np.zeros(nd, np.uint32)
            _check(self.L.cb_download_block(self._h, 0, l, p(dst), p(src), p(edges), p(dpos)))
            out.blocks.append({"layer": l, "dst": dst, "src": src, "edges": edges,
                               "dst_pos": dpos})
            n_src, n_own = C.c_uint64(), C.c_uint64()
            _check(self.L.cb_px_sizes(self._h, l, C.byref(n_src), C.byref(n_own)))
            send = np.zeros(self.world, np.uint64)
            lp, lr = np.zeros(n_src.value, np.uint32), np.zeros(n_src.value, np.uint32)
            own = np.zeros(n_own.value, np.uint32)
            _check(self.L.cb_px_download(self._h, l, p(send), p(lp), p(lr), p(own)))
            out.exchanges.append(DistExchange(l, [int(x) for x in send], n_own.value, lp,
                                              lr.astype(np.uint64)))
            out.owner_set = own
        return out

    def rows(self) -> np.ndarray:
        n = C.c_uint64()
        _check(self.L.cb_px_sizes(self._h, self.num_layers - 1, C.byref(n), None))
        dt = _DT[self.store.dtype][1]
        out = np.zeros((n.value, self.store.dim), dtype=dt)
        _check(self.L.cb_download_rows(self._h, 0, out.ctypes.data_as(C.c_void_p)))
        return out
