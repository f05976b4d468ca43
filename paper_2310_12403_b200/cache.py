"""Host mirror of the reference's cache API (proj/include/coopbatch/cache.hpp)
over the device LRU of libcoopbatch_b200 (csrc/cache.cu).

* ``LruCache``                 <- LruCache (cache.hpp:17-42, cache.cpp:8-32)
* ``feature_load_sim``         <- feature_load_sim (cache.hpp:80-83, cache.cpp:88-119)
* ``run_dependent_experiment`` <- run_dependent_experiment (cache.hpp:101-108,
                                  cache.cpp:137-208)
* ``nested_batches``           <- nested_batches (cache.hpp:62-66, cache.cpp:34-66)
* ``stack_fingerprint``        <- the fingerprint of cache.cpp:123-133

Hit/miss decisions are exact LRU (the device evaluates one id set per call,
see cache.h); the experiment driver samples every step on the GPU and, given a
FeatureStore, moves the rows too: hits from the cache's HBM rows, misses from
the table (HBM or the pinned host tier, ``FeatureStore.set_tier``).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .coopbatch import (KAPPA_INFINITY, MODE_INDEP, FeatureStore, Graph, InputError,
                        LayerStack, PartitionMap, Plan, SamplerConfig, SeedSchedule, _check,
                        _ptr, expand, hash_bits, schedule_advance)


class CacheOutcome(enum.IntEnum):  # cache.hpp:14
    kHit = 0
    kMiss = 1


class BatchMode(enum.IntEnum):  # cache.hpp:44
    kIndependent = 0
    kNested = 1
    kSmoothed = 2


@dataclass
class MinibatchSchedule:  # cache.hpp:50-54
    mode: BatchMode = BatchMode.kIndependent
    kappa: int = 1
    batch_size: int = 1024


@dataclass
class CacheStats:  # cache.hpp:68-74
    hits: int = 0
    misses: int = 0
    accesses: int = 0
    miss_rate: float = 0.0
    bytes: int = 0


@dataclass
class DependentStepRow:  # cache.hpp:85-91
    step: int = 0
    miss_rate: float = 0.0
    s_l: int = 0
    bytes: int = 0
    fingerprint: int = 0


@dataclass
class DependentExperimentResult:  # cache.hpp:93-98
    rows: list[DependentStepRow] = field(default_factory=list)
    warmup_steps: int = 0
    steps_per_epoch: int = 0
    steady_miss_rate: float = 0.0


class ClockCache:
    """Set-associative feature cache with CLOCK replacement (cb_ccache_*): the
    fast production mode. Three kernels per batch, no sort and no host round
    trip; its hit rate is its own (LruCache is the batch-exact LRU for parity),
    and the rows it serves are always the table's rows."""

    def __init__(self, capacity: int, row_bytes: int, device: int = 0, ways: int = 8):
        if capacity < 1:
            raise InputError("ClockCache: capacity must be >= 1")
        h = C.c_void_p()
        _check(_lib.load().cb_ccache_create(device, capacity, ways, row_bytes, C.byref(h)))
        self._h = h

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                _lib.load().cb_ccache_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown: the loader may be gone
            pass

    def gather_plan(self, plan: Plan, part: int, store: FeatureStore):
        """Input rows of `part` of the plan's last batch into the plan's row
        buffer (Plan.rows): hits from the cache, misses from `store`."""
        _check(_lib.load().cb_ccache_gather_plan(self._h, plan._h, part, store._h))

    def stats(self) -> tuple[int, int, int]:
        """(hits, inserted rows, slots) so far."""
        h, i, s = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(_lib.load().cb_ccache_stats(self._h, C.byref(h), C.byref(i), C.byref(s)))
        return h.value, i.value, s.value


class LruCache:
    """Exact LRU over vertex ids [0, n_keys), resident on `device`. With
    row_bytes > 0 it also holds the rows of its resident keys in HBM."""

    def __init__(self, capacity: int, n_keys: int, device: int = 0, row_bytes: int = 0):
        if capacity < 1:
            raise InputError("LruCache: capacity must be >= 1")
        h = C.c_void_p()
        _check(_lib.load().cb_cache_create(device, n_keys, capacity, row_bytes, C.byref(h)))
        self._h, self.n_keys, self._cap = h, n_keys, capacity

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                _lib.load().cb_cache_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown: the loader may be gone
            pass

    def capacity(self) -> int:
        return self._cap

    def _stats(self):
        h, m, s = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(_lib.load().cb_cache_stats(self._h, C.byref(h), C.byref(m), C.byref(s)))
        return h.value, m.value, s.value

    def hits(self) -> int:
        return self._stats()[0]

    def misses(self) -> int:
        return self._stats()[1]

    def size(self) -> int:
        return self._stats()[2]

    def miss_rate(self) -> float:
        h, m, _ = self._stats()
        return 0.0 if h + m == 0 else m / (h + m)

    def reset_counters(self):
        _check(_lib.load().cb_cache_reset_counters(self._h))

    def access(self, key: int) -> CacheOutcome:
        return CacheOutcome(int(self.access_trace([key])[0]))

    def access_trace(self, keys) -> np.ndarray:
        """LruCache::access over the keys in order; 1 = miss."""
        k = np.ascontiguousarray(keys, dtype=np.uint32)
        miss = np.zeros(len(k), np.uint8)
        _check(_lib.load().cb_cache_access_trace(self._h, _ptr(k), len(k), _ptr(miss)))
        return miss

    def access_ids(self, ids, order_key: int, pm: PartitionMap | None = None,
                   part: int = 0) -> int:
        """One step of feature_load_sim for a sorted unique id list: access in
        access_order(ids, order_key), owned ids only when pm is given."""
        k = np.ascontiguousarray(ids, dtype=np.uint32)
        kept = C.c_uint64()
        _check(_lib.load().cb_cache_access_host_ids(self._h, _ptr(k), len(k), order_key,
                                                    pm._h if pm else None, part,
                                                    C.byref(kept)))
        return kept.value

    def access_plan(self, plan: Plan, part: int, order_key: int,
                    pm: PartitionMap | None = None, owner_part: int = 0,
                    store: FeatureStore | None = None) -> int:
        """Same over the device-resident input vertices of a sampled plan; with
        `store` the rows land in the plan's row buffer (Plan.rows)."""
        kept = C.c_uint64()
        _check(_lib.load().cb_cache_access_plan(self._h, plan._h, part, order_key,
                                                pm._h if pm else None, owner_part,
                                                store._h if store else None, None,
                                                C.byref(kept)))
        return kept.value

    def resident(self) -> np.ndarray:
        out = np.zeros(min(self._cap, self.n_keys), np.uint32)
        n = C.c_uint64()
        _check(_lib.load().cb_cache_resident(self._h, _ptr(out), len(out), C.byref(n)))
        return out[: n.value]


def lru_access(c: LruCache, key: int) -> CacheOutcome:  # cache.hpp:44
    return c.access(key)


def stack_fingerprint(plan: Plan, part: int = 0) -> int:
    """cache.cpp:123-133 over part `part` of the plan's last batch."""
    out = C.c_uint64()
    _check(_lib.load().cb_stack_fingerprint(plan._h, part, C.byref(out)))
    return out.value


def shuffled_order(n: int, seed: int) -> np.ndarray:
    """cache.cpp:155-162: the fixed training order of the dependent experiment."""
    out = np.zeros(n, np.uint32)
    _check(_lib.load().cb_shuffled_order(n, seed, _ptr(out)))
    return out


def feature_load_sim(steps: list[list[LayerStack]], caches: list[LruCache],
                     pm: PartitionMap | None, dim: int,
                     bytes_per_scalar: int) -> list[CacheStats]:
    """cache.cpp:88-119: every step's input vertices through per-PE caches
    (cooperative: owned ids only), ordered by access_order(ids,
    hash_bits(step_index, {p})) with step_index counted from 1."""
    parts = len(caches)
    for step in steps:
        if len(step) != parts:
            raise InputError("feature_load_sim: stack/cache count mismatch")
    base = [(c.hits(), c.misses()) for c in caches]
    acc = [0] * parts
    for si, step in enumerate(steps, start=1):
        for p in range(parts):
            acc[p] += caches[p].access_ids(step[p].input_vertices(), hash_bits(si, [p]), pm, p)
    out = []
    for p in range(parts):
        h, m = caches[p].hits() - base[p][0], caches[p].misses() - base[p][1]
        out.append(CacheStats(h, m, acc[p], 0.0 if acc[p] == 0 else m / acc[p],
                              m * dim * bytes_per_scalar))
    return out


def nested_batches(g: Graph, super_seeds, kappa: int, b: int, num_layers: int,
                   cfg: SamplerConfig, epoch_seed: int) -> list[LayerStack]:
    """cache.cpp:34-66: kappa b-sized slices of one super batch, each expanded
    under the super batch's epoch seed; layerwise containment is verified."""
    if kappa == 0 or b == 0:
        raise InputError("nested_batches: kappa and b must be >= 1")
    sup = np.ascontiguousarray(super_seeds, dtype=np.uint32)
    if len(sup) != kappa * b:
        raise InputError("nested_batches: super batch must hold exactly kappa*b seeds")
    sched = SeedSchedule.plain(epoch_seed)
    whole = expand(g, sup, num_layers, cfg, sched)
    stacks = [expand(g, sup[i * b:(i + 1) * b], num_layers, cfg, sched) for i in range(kappa)]
    for l in range(num_layers):
        for st in stacks:
            if not np.isin(st.blocks[l].src_vertices, whole.blocks[l].src_vertices).all():
                raise InputError(f"nested_batches: containment violated at layer {l}")
    return stacks


def run_dependent_experiment(g: Graph, schedule: MinibatchSchedule, steps: int,
                             cache_capacity: int, cfg: SamplerConfig, num_layers: int,
                             feature_dim: int, bytes_per_scalar: int, seed: int,
                             fingerprints: bool = True, store: FeatureStore | None = None,
                             on_step=None, cache_kind: str = "lru") -> DependentExperimentResult:
    """cache.cpp:137-208 on the GPU: a fixed shuffled order sliced into
    batches, each expanded under the schedule (smoothed kappa variates,
    nested groups or independent), its input rows fetched through the LRU.
    With `store` the rows really move (hits from the cache's HBM rows, misses
    from the store's tier). `on_step(step, plan)` is called after each step."""
    n = g.num_vertices
    b = min(schedule.batch_size, n)
    if b == 0:
        raise InputError("run_dependent_experiment: empty batches")
    order = shuffled_order(n, seed)
    spe = max(1, n // b)
    seeds = SeedSchedule.make(1 if schedule.mode == BatchMode.kNested else schedule.kappa, seed)
    if cache_kind not in ("lru", "clock"):
        raise InputError("run_dependent_experiment: cache_kind must be 'lru' or 'clock'")
    if cache_kind == "clock" and store is None:
        raise InputError("run_dependent_experiment: the CLOCK cache moves rows (give a store)")
    # "lru": the reference's LruCache decisions exactly; "clock": the fast
    # set-associative cache (its own hit rate, no per-step sort)
    cache = (LruCache(cache_capacity, n, g.device, store.row_bytes if store else 0)
             if cache_kind == "lru" else ClockCache(cache_capacity, store.row_bytes, g.device))
    plan = Plan(g, None, num_layers, cfg, b)
    res = DependentExperimentResult(steps_per_epoch=spe, warmup_steps=min(spe, steps // 2))
    steady_hits = steady_miss = 0
    for step in range(steps):
        slot = (step % spe) * b
        batch = order[slot:slot + b]
        if schedule.mode == BatchMode.kNested:
            group = 0 if schedule.kappa == KAPPA_INFINITY else step // schedule.kappa
            z = hash_bits(seed, [12, group])
            plan.sample([batch], SeedSchedule(1, z, z, 0), MODE_INDEP)
        else:
            plan.sample([batch], seeds, MODE_INDEP)
            seeds = schedule_advance(seeds)
        fp = stack_fingerprint(plan, 0) if fingerprints else 0
        if cache_kind == "lru":
            m0 = cache.misses()
            s_l = cache.access_plan(plan, 0, hash_bits(seed, [step, 0xACCE55]), store=store)
            miss = cache.misses() - m0
        else:
            h0 = cache.stats()[0]
            cache.gather_plan(plan, 0, store)
            s_l = plan.layer_sizes(0, num_layers - 1)["n_src"]
            miss = s_l - (cache.stats()[0] - h0)
        res.rows.append(DependentStepRow(step, 0.0 if s_l == 0 else miss / s_l, s_l,
                                         miss * feature_dim * bytes_per_scalar, fp))
        if step >= res.warmup_steps:
            steady_miss += miss
            steady_hits += s_l - miss
        if on_step:
            on_step(step, plan)
    tot = steady_hits + steady_miss
    res.steady_miss_rate = 0.0 if tot == 0 else steady_miss / tot
    return res
