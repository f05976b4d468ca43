"""Host-side mirror of the reference's sampler / minibatch API
(/root/reference/proj/include/coopbatch/{graph,rng,samplers,partition,coop}.hpp)
over the libcoopbatch_b200 C-ABI. Same names, argument meaning and error
behaviour (contract violations raise ``InputError``, the mirror of
``coopbatch::InputError``, common.hpp:12-15); results are returned by value
as numpy arrays, like the reference's ``std::vector`` value types.

All computation runs in the sm_100a kernels of ``libcoopbatch_b200.so``; this
module only marshals arguments and downloads results.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import Sched

KAPPA_INFINITY = (1 << 64) - 1  # rng.hpp:70-71

_MASK = (1 << 64) - 1
_SALT = 0x736F6D6570736575


class InputError(ValueError):
    """coopbatch::InputError (common.hpp:12-15)."""


class FormatError(RuntimeError):
    """coopbatch::FormatError (common.hpp:23-26)."""


class CudaError(RuntimeError):
    """CUDA / NCCL failure inside libcoopbatch_b200."""


class CapacityError(RuntimeError):
    """A device capacity bound overflowed (cb_sample_sync retries these)."""


class UncertifiedError(RuntimeError):
    """Smoothed variate decisions inside the guard band were left unresolved
    (an asynchronous path; cb_sample_sync resolves them on the host)."""


_ERRS = {1: InputError, 2: FormatError, 3: OSError, 4: CudaError, 5: CudaError,
         6: CapacityError, 7: RuntimeError, 8: UncertifiedError}


def _check(rc: int):
    if rc != 0:
        L = _lib.load()
        raise _ERRS.get(rc, RuntimeError)(L.cb_last_error().decode())


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ------------------------------------------------------------------- rng ----
def mix64(x: int) -> int:
    """rng.hpp:17-22 (host helper for seed draws / schedules)."""
    x = (x + 0x9E3779B97F4A7C15) & _MASK
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _MASK
    return x ^ (x >> 31)


def hash_bits(seed: int, ids) -> int:
    """rng.hpp:34-39."""
    h = mix64((seed ^ _SALT) & _MASK)
    for i in ids:
        h = mix64(h ^ (int(i) & _MASK))
    return h


def hash_uniform(seed: int, ids) -> float:
    return (hash_bits(seed, ids) >> 11) * 2.0 ** -53


class SamplerKind(enum.IntEnum):  # samplers.hpp:15
    kFull = 0
    kNs = 1
    kLabor0 = 2
    kRw = 3


@dataclass
class SamplerConfig:  # samplers.hpp:17-23 (+ per-layer fanouts extension)
    kind: SamplerKind = SamplerKind.kNs
    fanout: int = 10
    fanouts: list[int] | None = None  # fanouts[l] applies at block l
    rw_length: int = 3      # o (samplers.hpp:20-22)
    rw_restart: float = 0.5  # p
    rw_walks: int = 100     # a

    def layer_fanouts(self, num_layers: int) -> list[int]:
        if self.fanouts:
            if len(self.fanouts) != num_layers:
                raise InputError("fanouts must list one fanout per layer")
            return [int(f) for f in self.fanouts]
        return [int(self.fanout)] * num_layers


@dataclass
class SeedSchedule:  # rng.hpp:93-111
    kappa: int = 1
    z1: int = 0
    z2: int = 0
    iteration: int = 0

    @staticmethod
    def make(kappa: int, root_seed: int) -> "SeedSchedule":  # rng.cpp:69-77
        if kappa == 0:
            raise InputError("SeedSchedule: kappa must be >= 1 (or infinity)")
        return SeedSchedule(kappa, hash_bits(root_seed, [12, 1]),
                            hash_bits(root_seed, [12, 2]), 0)

    @staticmethod
    def plain(seed: int) -> "SeedSchedule":
        """kappa 1, z1 = z2 = seed (the reference tests' plain_schedule)."""
        return SeedSchedule(1, seed, seed, 0)

    def contribution(self) -> float:
        if self.kappa == KAPPA_INFINITY:
            return 0.0
        return (self.iteration % self.kappa) / self.kappa

    def smoothing_active(self) -> bool:
        return self.kappa != KAPPA_INFINITY and self.kappa >= 2

    def _c(self) -> Sched:
        return Sched(self.kappa, self.z1, self.z2, self.iteration)


def schedule_advance(s: SeedSchedule) -> SeedSchedule:  # rng.cpp:79-86
    t = SeedSchedule(s.kappa, s.z1, s.z2, s.iteration + 1)
    if t.kappa != KAPPA_INFINITY and t.iteration % t.kappa == 0:
        t.z1 = t.z2
        t.z2 = hash_bits(t.z2, [12, t.iteration])
    return t


# ----------------------------------------------------------------- graph ----
class Graph:
    """coopbatch::Graph (graph.hpp:21-53): in-neighbour CSR resident in HBM."""

    def __init__(self, handle, device: int):
        self._h = handle
        self.device = device
        L = _lib.load()
        n, m, md = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(L.cb_graph_info(self._h, C.byref(n), C.byref(m), C.byref(md)))
        self.num_vertices, self._m, self.max_degree = n.value, m.value, md.value

    @classmethod
    def from_csr(cls, indptr, indices, device: int = 0, weights=None) -> "Graph":
        """weights: one positive float per edge (graph.hpp:25), read by the RW
        sampler's weighted neighbour pick."""
        indptr = np.ascontiguousarray(indptr, dtype=np.uint64)
        indices = np.ascontiguousarray(indices, dtype=np.uint32)
        L = _lib.load()
        h = C.c_void_p()
        _check(L.cb_graph_create_from_csr(_ptr(indptr), _ptr(indices), len(indptr) - 1,
                                          len(indices), device, C.byref(h)))
        g = cls(h, device)
        if weights is not None:
            w = np.ascontiguousarray(weights, dtype=np.float32)
            if len(w) != len(indices):
                raise InputError("weights must have one entry per edge")
            _check(L.cb_graph_set_weights(g._h, _ptr(w)))
        return g

    @classmethod
    def generate_rmat(cls, num_vertices: int, num_edges: int, seed: int,
                      device: int = 0) -> "Graph":
        """Hash-keyed R-MAT built on the device (DESIGN.md §Synthetic graph)."""
        L = _lib.load()
        h = C.c_void_p()
        _check(L.cb_graph_generate_rmat(num_vertices, num_edges, seed, device, C.byref(h)))
        return cls(h, device)

    def num_edges(self) -> int:
        return self._m

    @classmethod
    def load_csr(cls, path: str, device: int = 0) -> "Graph":
        """load_csr (graph.cpp:231-252): a CBCS file straight into HBM."""
        h = C.c_void_p()
        _check(_lib.load().cb_graph_load_cbcs(str(path).encode(), device, C.byref(h)))
        return cls(h, device)

    def save_csr(self, path: str):
        """save_csr (graph.cpp:216-229)."""
        _check(_lib.load().cb_graph_save_cbcs(self._h, str(path).encode()))

    def download(self):
        indptr = np.zeros(self.num_vertices + 1, np.uint64)
        indices = np.zeros(self._m, np.uint32)
        _check(_lib.load().cb_graph_download(self._h, _ptr(indptr), _ptr(indices)))
        return indptr, indices

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                _lib.load().cb_graph_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown: the loader may be gone
            pass


class PartitionMap:
    """coopbatch::PartitionMap (partition.hpp:12-17), resident on the device."""

    def __init__(self, g: Graph, handle, parts: int):
        self._g = g
        self._h = handle
        self.num_parts = parts

    @property
    def owner(self) -> np.ndarray:
        o = np.zeros(self._g.num_vertices, np.uint32)
        _check(_lib.load().cb_partition_download(self._h, _ptr(o)))
        return o

    def members(self) -> list[np.ndarray]:
        """part_members (partition.cpp:99-105): ascending members of each part."""
        m = np.zeros(self._g.num_vertices, np.uint32)
        off = np.zeros(self.num_parts + 1, np.uint64)
        _check(_lib.load().cb_partition_members(self._h, _ptr(m), _ptr(off)))
        return [m[int(off[q]):int(off[q + 1])] for q in range(self.num_parts)]

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                _lib.load().cb_partition_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown: the loader may be gone
            pass


def partition_random(g: Graph, parts: int, seed: int) -> PartitionMap:
    """partition.cpp:10-20 — owner(v) = hash(seed, {7, v}) mod parts."""
    h = C.c_void_p()
    _check(_lib.load().cb_partition_random(g._h, parts, seed, C.byref(h)))
    return PartitionMap(g, h, parts)


def cross_edge_ratio(g: Graph, pm: PartitionMap) -> float:
    """partition.cpp:79-89 — fraction of edges whose endpoints have different owners."""
    r = C.c_double()
    _check(_lib.load().cb_cross_edge_ratio(g._h, pm._h, None, C.byref(r)))
    return r.value


def partition_from_owner(g: Graph, owner, parts: int) -> PartitionMap:
    owner = np.ascontiguousarray(owner, dtype=np.uint32)
    if len(owner) != g.num_vertices:
        raise InputError("partition: owner array does not cover all vertices")
    h = C.c_void_p()
    _check(_lib.load().cb_partition_create(g._h, _ptr(owner), parts, C.byref(h)))
    return PartitionMap(g, h, parts)


_DT = {"f64": (0, np.float64), "f32": (1, np.float32), "f16": (2, np.float16)}


class FeatureStore:
    """coopbatch::FeatureStore (coop.hpp:140-155): synthetic rows, one
    rounding to `dtype`, row-sharded by `pm` (rows of part q = its members in
    ascending id order)."""

    def __init__(self, g: Graph, handle, dim: int, dtype: str, pm: PartitionMap | None):
        self._g, self._h, self.dim, self.dtype, self._pm = g, handle, dim, dtype, pm
        self.row_bytes = dim * np.dtype(_DT[dtype][1]).itemsize

    @classmethod
    def synth(cls, g: Graph, dim: int, seed: int, dtype: str = "f32",
              pm: PartitionMap | None = None) -> "FeatureStore":
        h = C.c_void_p()
        _check(_lib.load().cb_features_synth(g._h, pm._h if pm else None, dim, _DT[dtype][0],
                                             seed, C.byref(h)))
        return cls(g, h, dim, dtype, pm)

    def set_tier(self, host: bool):
        """Move the table to pinned host memory mapped into the device (the
        paper's storage channel: every row read crosses the host link) or back
        to HBM. Rows and their layout are unchanged."""
        _check(_lib.load().cb_features_set_tier(self._h, int(bool(host))))

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                _lib.load().cb_features_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown: the loader may be gone
            pass


# ---------------------------------------------------------------- results ---
@dataclass
class BipartiteBlock:  # samplers.hpp:30-38
    dst_vertices: np.ndarray
    src_vertices: np.ndarray
    edges: np.ndarray  # (n_edges, 2) u32 (src_idx, dst_idx)
    dst_pos_in_src: np.ndarray
    layer: int = 0
    uncertified: int = 0

    def num_edges(self) -> int:
        return len(self.edges)

    def as_dict(self) -> dict:
        return {"layer": self.layer, "dst": self.dst_vertices, "src": self.src_vertices,
                "edges": self.edges, "dst_pos": self.dst_pos_in_src}


@dataclass
class LayerStack:  # samplers.hpp:42-49
    blocks: list[BipartiteBlock] = field(default_factory=list)

    def input_vertices(self) -> np.ndarray:
        return self.blocks[-1].src_vertices


@dataclass
class ExchangeRecord:  # coop.hpp:25-37
    layer: int
    send_counts: np.ndarray       # (P, P)
    owner_row_counts: np.ndarray  # (P,)
    loc_part: list[np.ndarray]
    loc_row: list[np.ndarray]

    def num_parts(self) -> int:
        return len(self.owner_row_counts)

    def communicated(self, p: int) -> int:  # coop.cpp:10-15
        return int(self.send_counts[p].sum() - self.send_counts[p, p])

    def total_communicated(self) -> int:
        return sum(self.communicated(p) for p in range(self.num_parts()))


@dataclass
class CoopSampleResult:  # coop.hpp:39-43
    stacks: list[LayerStack]
    exchanges: list[ExchangeRecord]
    owner_sets: list[np.ndarray]


# ------------------------------------------------------------------ plans ---
MODE_COOP, MODE_INDEP = 0, 1


class Plan:
    """A cb_plan: device workspace for one (graph, partition, L, sampler)
    combination; reusable across batches."""

    def __init__(self, g: Graph, pm: PartitionMap | None, num_layers: int,
                 cfg: SamplerConfig, max_seeds_per_part: int, parts: int | None = None):
        """parts (with pm None): that many independent parts without a
        partition (indep mode only; cb_plan_create_parts)."""
        self.g, self.pm, self.L, self.cfg = g, pm, num_layers, cfg
        self.max_seeds = max_seeds_per_part
        fo = np.asarray(cfg.layer_fanouts(num_layers), dtype=np.uint32)
        h = C.c_void_p()
        if pm is None and parts is not None:
            _check(_lib.load().cb_plan_create_parts(g._h, parts, num_layers, int(cfg.kind),
                                                    _ptr(fo), max_seeds_per_part, C.byref(h)))
        else:
            _check(_lib.load().cb_plan_create(g._h, pm._h if pm else None, num_layers,
                                              int(cfg.kind), _ptr(fo), max_seeds_per_part,
                                              C.byref(h)))
        self._h = h
        if cfg.kind == SamplerKind.kRw:
            _check(_lib.load().cb_plan_set_rw(h, cfg.rw_length, cfg.rw_restart, cfg.rw_walks))
        self.P = pm.num_parts if pm else (parts or 1)

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                _lib.load().cb_plan_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown: the loader may be gone
            pass

    @property
    def stream(self) -> int:
        return int(_lib.load().cb_plan_stream(self._h) or 0)

    @staticmethod
    def _flat(per_pe_seeds):
        arrs = [np.ascontiguousarray(s, dtype=np.uint32) for s in per_pe_seeds]
        off = np.zeros(len(arrs) + 1, np.uint64)
        off[1:] = np.cumsum([len(a) for a in arrs])
        flat = np.concatenate(arrs) if arrs else np.zeros(0, np.uint32)
        return np.ascontiguousarray(flat, dtype=np.uint32), off

    def sample(self, per_pe_seeds, schedule: SeedSchedule, mode: int = MODE_COOP,
               sync: bool = True):
        if len(per_pe_seeds) != self.P:
            raise InputError("coop_sample: seed lists must match the partition count")
        flat, off = self._flat(per_pe_seeds)
        self._keep = (flat, off)
        s = schedule._c()
        f = _lib.load().cb_sample_sync if sync else _lib.load().cb_sample
        _check(f(self._h, mode, _ptr(flat), _ptr(off), C.byref(s)))

    def sample_multi(self, per_pe_seeds, schedules: list[SeedSchedule]):
        """Independent expansions, part p under schedules[p] (cb_sample_multi)."""
        if len(per_pe_seeds) != self.P or len(schedules) != self.P:
            raise InputError("sample_multi: one seed list and one schedule per part")
        flat, off = self._flat(per_pe_seeds)
        self._keep = (flat, off)
        sc = (Sched * self.P)(*[s._c() for s in schedules])
        _check(_lib.load().cb_sample_multi(self._h, _ptr(flat), _ptr(off), sc))

    def sample_device(self, d_seeds_ptr: int, offsets, schedule: SeedSchedule,
                      mode: int = MODE_COOP):
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        s = schedule._c()
        _check(_lib.load().cb_sample_device(self._h, mode, C.c_void_p(d_seeds_ptr),
                                            _ptr(off), C.byref(s)))

    def capture(self, offsets, schedule: SeedSchedule, mode: int = MODE_COOP,
                store: FeatureStore | None = None):
        """Capture one batch (and its gather) as CUDA graphs for replay."""
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        s = schedule._c()
        _check(_lib.load().cb_plan_capture(self._h, mode, _ptr(off),
                                           store._h if store else None, C.byref(s)))

    def replay(self, seeds_ptr: int | None, schedule: SeedSchedule | None,
               on_device: bool, what: int = 3):
        s = schedule._c() if schedule is not None else None
        _check(_lib.load().cb_plan_replay(self._h, C.c_void_p(seeds_ptr) if seeds_ptr else None,
                                          int(on_device), C.byref(s) if s is not None else None,
                                          what))

    def gather(self, store: FeatureStore):
        _check(_lib.load().cb_gather(self._h, store._h))

    def synchronize(self):
        _check(_lib.load().cb_synchronize(self._h))

    def set_guard(self, band: float = 1e-12, perturb: bool = False, strict: bool = True):
        """Guard band of smoothed decisions (cb_plan_set_guard): in-band decisions
        are resolved on the host with the reference's arithmetic by the
        synchronous sample; `perturb` flips unresolved in-band device decisions
        (a test hook for the re-sampling path)."""
        _check(_lib.load().cb_plan_set_guard(self._h, band, int(perturb), int(strict)))

    def resolve_stats(self) -> tuple[int, int]:
        """(decisions resolved on the host, re-samplings) of the last sync sample."""
        a, b = C.c_uint64(), C.c_uint64()
        _check(_lib.load().cb_plan_resolve_stats(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def profile(self, per_pe_seeds, schedule: SeedSchedule, mode: int = MODE_COOP,
                store: FeatureStore | None = None) -> list[float]:
        """Per-launch device times (ms) of one eager batch, enqueue order."""
        flat, off = self._flat(per_pe_seeds)
        ms = np.zeros(256, np.float32)
        n = C.c_int()
        s = schedule._c()
        _check(_lib.load().cb_plan_profile(self._h, mode, _ptr(flat), _ptr(off), C.byref(s),
                                           store._h if store else None, _ptr(ms), 256,
                                           C.byref(n)))
        return ms[: n.value].tolist()

    def graph_profile(self, seeds_ptr: int | None, schedule: SeedSchedule) -> list[float]:
        """In-graph per-launch device times (ms) of one replay of the captured batch."""
        ms = np.zeros(256, np.float32)
        n = C.c_int()
        s = schedule._c()
        _check(_lib.load().cb_plan_graph_profile(self._h, C.c_void_p(seeds_ptr) if seeds_ptr
                                                 else None, C.byref(s), _ptr(ms), 256,
                                                 C.byref(n)))
        return ms[: n.value].tolist()

    def captured_launches(self, what: int = 3) -> int:
        """Kernels per replay of the captured graph (1 sample, 2 gather, 3 both)."""
        n = C.c_uint64()
        _check(_lib.load().cb_plan_captured_launches(self._h, what, C.byref(n)))
        return n.value

    def launch_count(self, mode: int, with_gather: bool) -> int:
        n = C.c_uint64()
        _check(_lib.load().cb_plan_launch_count(self._h, mode, int(with_gather), C.byref(n)))
        return n.value

    def all_layer_sizes(self) -> np.ndarray:
        """All parts' per-layer counts in one read: [P, L+1, 8] u64 records
        (n_dst, scan_total, n_active, n_edges, n_src, uncertified, pad, pad)."""
        L = _lib.load()
        nb = C.c_uint64()
        _check(L.cb_plan_meta_async(self._h, None, C.byref(nb)))
        out = np.zeros(nb.value // 8, np.uint64)
        _check(L.cb_plan_meta_async(self._h, _ptr(out), None))
        self.synchronize()
        return out.reshape(self.P, self.L + 1, 8)

    def layer_sizes(self, p: int, l: int) -> dict:
        s = np.zeros(6, np.uint64)
        _check(_lib.load().cb_layer_sizes(self._h, p, l, _ptr(s)))
        return {"n_dst": int(s[0]), "n_src": int(s[1]), "n_edges": int(s[2]),
                "uncertified": int(s[3]), "scan_total": int(s[4]), "n_active": int(s[5])}

    def block(self, p: int, l: int) -> BipartiteBlock:
        sz = self.layer_sizes(p, l)
        dst = np.zeros(sz["n_dst"], np.uint32)
        src = np.zeros(sz["n_src"], np.uint32)
        edges = np.zeros((sz["n_edges"], 2), np.uint32)
        dpos = np.zeros(sz["n_dst"], np.uint32)
        _check(_lib.load().cb_download_block(self._h, p, l, _ptr(dst), _ptr(src), _ptr(edges),
                                             _ptr(dpos)))
        return BipartiteBlock(dst, src, edges, dpos, l, sz["uncertified"])

    def stack(self, p: int) -> LayerStack:
        return LayerStack([self.block(p, l) for l in range(self.L)])

    def owner_set(self, p: int) -> np.ndarray:
        n = C.c_uint64()
        L = _lib.load()
        _check(L.cb_owner_set_size(self._h, p, C.byref(n)))
        ids = np.zeros(n.value, np.uint32)
        _check(L.cb_download_owner_set(self._h, p, _ptr(ids)))
        return ids

    def exchange(self, l: int) -> ExchangeRecord:
        P = self.P
        lens = [self.layer_sizes(p, l)["n_src"] for p in range(P)]
        sc = np.zeros((P, P), np.uint64)
        orc = np.zeros(P, np.uint64)
        lp = np.zeros(sum(lens), np.uint32)
        lr = np.zeros(sum(lens), np.uint64)
        _check(_lib.load().cb_download_exchange(self._h, l, _ptr(sc), _ptr(orc), _ptr(lp),
                                                _ptr(lr)))
        offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        return ExchangeRecord(l, sc, orc, [lp[offs[p]:offs[p + 1]] for p in range(P)],
                              [lr[offs[p]:offs[p + 1]] for p in range(P)])

    def result_bytes(self, p: int = 0, row_bytes: int = 0) -> int:
        n = C.c_uint64()
        _check(_lib.load().cb_plan_result_bytes(self._h, p, row_bytes, C.byref(n)))
        return n.value

    def result_async(self, host_ptr: int, cap: int, p: int = 0):
        """Part p's blocks (+ gathered rows) into pinned host memory at
        host_ptr, ordered on the plan stream (parse_result reads it)."""
        _check(_lib.load().cb_plan_result_async(self._h, p, C.c_void_p(host_ptr), cap))

    def result_pack(self, p: int = 0):
        """Pack the batch's result on the device, asynchronously (for result_copy)."""
        _check(_lib.load().cb_plan_result_pack(self._h, p))

    def result_copy(self, host_ptr: int, cap: int, p: int = 0) -> int:
        """Same layout through a copy engine (cb_plan_result_copy): waits for the
        batch and its pack, then enqueues one D2H copy; returns the size."""
        n = C.c_uint64()
        _check(_lib.load().cb_plan_result_copy(self._h, p, C.c_void_p(host_ptr), cap,
                                               C.byref(n)))
        return n.value

    def rows(self, p: int, store: FeatureStore) -> np.ndarray:
        n = self.layer_sizes(p, self.L - 1)["n_src"]
        out = np.zeros((n, store.dim), dtype=_DT[store.dtype][1])
        _check(_lib.load().cb_download_rows(self._h, p, _ptr(out)))
        return out


def parse_result(buf: np.ndarray, dtype=None, dim: int = 0) -> dict:
    """Reads a cb_plan_result_async buffer (csrc/result.cu layout): the
    per-layer blocks as dicts (dst, src, edges, dst_pos) and the rows."""
    b = np.asarray(buf).view(np.uint8)
    hd = b[:40].view(np.uint64)
    if int(hd[0]) != 0x3153524243:
        raise ValueError("not a batch result buffer")
    L, row_bytes, total, trunc = (int(x) for x in hd[1:5])
    if trunc:
        raise ValueError(f"result truncated: {total} bytes needed")
    cnt = b[40:40 + 24 * L].view(np.uint64).reshape(L, 3)
    pad = lambda x: (x + 15) & ~15  # noqa: E731
    off = pad(8 * (5 + 3 * L))
    out = {"blocks": []}

    def take(nbytes, dt):
        nonlocal off
        a = b[off:off + nbytes].view(dt)
        off += pad(nbytes)
        return a
    for l in range(L):
        nd, ns, ne = (int(x) for x in cnt[l])
        blk = {"layer": l, "dst": take(4 * nd, np.uint32), "src": take(4 * ns, np.uint32),
               "edges": take(8 * ne, np.uint32).reshape(ne, 2),
               "dst_pos": take(4 * nd, np.uint32)}
        out["blocks"].append(blk)
    if row_bytes:
        n = int(cnt[L - 1][1])
        raw = take(n * row_bytes, np.uint8)
        out["rows"] = raw.view(dtype).reshape(n, -1) if dtype is not None else raw
    out["total_bytes"] = total
    return out


# Plans of the reference-style free functions, most recently used last. A plan
# keeps its graph (and partition) alive, so the cache is bounded.
_plan_cache: dict = {}
_PLAN_CACHE_MAX = 16


def _plan_for(g: Graph, pm, num_layers: int, cfg: SamplerConfig, n_seeds: int) -> Plan:
    key = (id(g), id(pm) if pm else None, num_layers, int(cfg.kind),
           tuple(cfg.layer_fanouts(num_layers)), cfg.rw_length, cfg.rw_restart, cfg.rw_walks)
    pl = _plan_cache.pop(key, None)
    if pl is None or pl.max_seeds < n_seeds or pl.g is not g or pl.pm is not pm:
        pl = Plan(g, pm, num_layers, cfg, max(n_seeds, 1))
    _plan_cache[key] = pl
    while len(_plan_cache) > _PLAN_CACHE_MAX:
        _plan_cache.pop(next(iter(_plan_cache)))
    return pl


def clear_plan_cache():
    _plan_cache.clear()


# ---------------------------------------------------------- reference API ---
def expand(g: Graph, seeds, num_layers: int, cfg: SamplerConfig,
           schedule: SeedSchedule) -> LayerStack:
    """samplers.cpp:340-354 — L-layer expansion of one seed list."""
    if num_layers < 1:
        raise InputError("expand: num_layers must be >= 1")
    seeds = np.ascontiguousarray(seeds, dtype=np.uint32)
    pl = _plan_for(g, None, num_layers, cfg, len(seeds))
    pl.sample([seeds], schedule, MODE_INDEP)
    return pl.stack(0)


def sample_block(g: Graph, seeds, cfg: SamplerConfig, schedule: SeedSchedule,
                 layer: int = 0) -> BipartiteBlock:
    """samplers.cpp:323-338: one block of any sampler at layer `layer` (the
    layer namespaces the variates): a 1-layer plan whose block hashes as
    `layer` (cb_plan_set_layer_base)."""
    if layer < 0:
        raise InputError("sample_block: layer must be >= 0")
    seeds = np.ascontiguousarray(seeds, dtype=np.uint32)
    pl = Plan(g, None, 1, cfg, max(len(seeds), 1))
    _check(_lib.load().cb_plan_set_layer_base(pl._h, layer))
    pl.sample([seeds], schedule, MODE_INDEP)
    b = pl.block(0, 0)
    b.layer = layer
    return b


def sample_ns(g: Graph, seeds, k: int, epoch_seed: int, layer: int = 0) -> BipartiteBlock:
    """samplers.cpp:298-303."""
    if k == 0:
        raise InputError("sample_ns: fanout must be >= 1")
    if layer == 0:
        return expand(g, seeds, 1, SamplerConfig(SamplerKind.kNs, k),
                      SeedSchedule.plain(epoch_seed)).blocks[0]
    return sample_block(g, seeds, SamplerConfig(SamplerKind.kNs, k),
                        SeedSchedule.plain(epoch_seed), layer)


def sample_labor0(g: Graph, seeds, k: int, variate, layer: int = 0) -> BipartiteBlock:
    """samplers.cpp:305-312 (labor_block, samplers.cpp:89-104): LABOR-0 with a
    caller variate r(t): keep t -> s iff r(t) <= k / d_s. `variate` is a
    callable VertexId -> float (evaluated once per distinct neighbour of the
    seeds, on the host) or an array of num_vertices floats. The block is
    sampled on the GPU from that table (cb_plan_set_variate_table)."""
    if k < 1:
        raise InputError("sample_labor0: fanout must be >= 1")
    seeds = np.ascontiguousarray(seeds, dtype=np.uint32)
    n = g.num_vertices
    if callable(variate):
        table = np.zeros(n, np.float64)
        for t in sample_full(g, seeds).src_vertices.tolist():
            table[t] = float(variate(t))
    else:
        table = np.ascontiguousarray(variate, dtype=np.float64)
        if table.shape != (n,):
            raise InputError("sample_labor0: variate table must hold one value per vertex")
    pl = Plan(g, None, 1, SamplerConfig(SamplerKind.kLabor0, k), max(len(seeds), 1))
    _check(_lib.load().cb_plan_set_variate_table(pl._h, _ptr(table), 0))
    pl.sample([seeds], SeedSchedule.plain(0), MODE_INDEP)
    b = pl.block(0, 0)
    b.layer = layer
    return b


def sample_rw(g: Graph, seeds, cfg: SamplerConfig, epoch_seed: int,
              layer: int = 0) -> BipartiteBlock:
    """samplers.cpp:314-321: random walks with restart, top-k visits."""
    if cfg.rw_length < 1 or cfg.rw_walks < 1:
        raise InputError("sample_rw: rw_length and rw_walks must be >= 1")
    rcfg = SamplerConfig(SamplerKind.kRw, cfg.fanout, None, cfg.rw_length, cfg.rw_restart,
                         cfg.rw_walks)
    if layer == 0:
        return expand(g, seeds, 1, rcfg, SeedSchedule.plain(epoch_seed)).blocks[0]
    return sample_block(g, seeds, rcfg, SeedSchedule.plain(epoch_seed), layer)


def sample_full(g: Graph, seeds, layer: int = 0) -> BipartiteBlock:
    """samplers.cpp:289-296."""
    b = expand(g, seeds, 1, SamplerConfig(SamplerKind.kFull, 1), SeedSchedule.plain(0)).blocks[0]
    b.layer = layer
    return b


def indep_sample(g: Graph, per_pe_seeds, num_layers: int, cfg: SamplerConfig,
                 schedule: SeedSchedule) -> list[LayerStack]:
    """coop.cpp:108-119 — each part expands its own seeds, no exchange."""
    return [expand(g, s, num_layers, cfg, schedule) for s in per_pe_seeds]


def coop_sample(g: Graph, pm: PartitionMap, per_pe_seeds, num_layers: int,
                cfg: SamplerConfig, schedule: SeedSchedule) -> CoopSampleResult:
    """coop.cpp:68-106 — cooperative expansion with per-layer owner exchange."""
    if len(per_pe_seeds) != pm.num_parts:
        raise InputError("coop_sample: seed lists must match the partition count")
    if num_layers < 1:
        raise InputError("coop_sample: num_layers must be >= 1")
    n = max((len(s) for s in per_pe_seeds), default=1)
    pl = _plan_for(g, pm, num_layers, cfg, n)
    pl.sample(per_pe_seeds, schedule, MODE_COOP)
    return CoopSampleResult([pl.stack(p) for p in range(pl.P)],
                            [pl.exchange(l) for l in range(num_layers)],
                            [pl.owner_set(p) for p in range(pl.P)])


@dataclass
class LayerMetrics:  # coop.hpp:157-162
    s_l: int = 0            # |S^l_p| (block destinations)
    s_tilde_l: int = 0      # |S~^{l+1}_p| (block sources)
    e_l: int = 0            # |E^l_p|
    comm_vertices: int = 0  # ids this part sent away at this layer


@dataclass
class PeMetrics:  # coop.hpp:164-168
    layers: list[LayerMetrics] = field(default_factory=list)
    feat_bytes: int = 0
    input_rows: int = 0


def step_metrics(plan: Plan, mode: int, row_bytes: int) -> list[PeMetrics]:
    """The per-PE metrics coop_train_step / indep_train_step report
    (block_metrics, coop.cpp:428-434; comm_vertices = ExchangeRecord::
    communicated, coop.cpp:543-546; feat_bytes / input_rows from the rows each
    part loads: its owner set when cooperative, coop.cpp:456-460, its input
    vertices when independent, coop.cpp:579-581), read from the device counts
    of the plan's last batch."""
    out = []
    coop = mode == MODE_COOP and plan.P > 1
    ex = [plan.exchange(l) for l in range(plan.L)] if coop else None
    for p in range(plan.P):
        pm_ = PeMetrics()
        for l in range(plan.L):
            sz = plan.layer_sizes(p, l)
            pm_.layers.append(LayerMetrics(sz["n_dst"], sz["n_src"], sz["n_edges"],
                                           ex[l].communicated(p) if coop else 0))
        n = C.c_uint64()
        if coop:
            _check(_lib.load().cb_owner_set_size(plan._h, p, C.byref(n)))
            pm_.input_rows = n.value
        else:
            pm_.input_rows = pm_.layers[-1].s_tilde_l
        pm_.feat_bytes = pm_.input_rows * row_bytes
        out.append(pm_)
    return out


def load_inputs(g: Graph, pm: PartitionMap | None, per_pe_seeds, num_layers: int,
                cfg: SamplerConfig, schedule: SeedSchedule, store: FeatureStore,
                mode: int = MODE_COOP) -> list[np.ndarray]:
    """Sample, then gather every part's input-feature rows requester-aligned:
    the composition all_to_all_forward(rec_{L-1}, load_rows(owner_sets))
    (coop.cpp:457-467), fused on the device."""
    n = max((len(s) for s in per_pe_seeds), default=1)
    pl = _plan_for(g, pm, num_layers, cfg, n)
    pl.sample(per_pe_seeds, schedule, mode)
    pl.gather(store)
    return [pl.rows(p, store) for p in range(pl.P)]
