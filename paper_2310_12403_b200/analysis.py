"""Work curves and the concavity check of the reference's analysis layer
(proj/include/coopbatch/analysis.hpp:13-45, proj/src/analysis.cpp:15-151),
with the trials sampled on the GPU.

* ``work_curve``      <- work_curve (analysis.cpp:78-124). Every trial draws
  its seeds on the host exactly as the reference does, then expands under
  its own fresh plain stream hash_bits(seed, {tag, 9}). The trials of one
  batch size run as the independent parts of ONE plan (cb_sample_multi):
  one launch sequence per ``trials_per_launch`` trials, parts on concurrent
  streams, instead of one expansion per trial.
* ``concavity_check`` <- concavity_check (analysis.cpp:126-151), host math.

Results equal the reference's: |S^L| per trial is bit-exact (integer
sampling path), and mean / standard error are summed in trial order as the
reference does.
"""
from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field

import numpy as np

from .coopbatch import Graph, InputError, Plan, SamplerConfig, SeedSchedule, hash_bits
from .seeds import edge_pred_seeds, first_distinct


class SeedMode(enum.IntEnum):  # analysis.hpp:28
    kNode = 0
    kEdge = 1


@dataclass
class WorkCurvePoint:  # analysis.hpp:15-21
    batch_size: int = 0
    mean_sl: float = 0.0
    se_sl: float = 0.0
    work_per_seed: float = 0.0
    se_work: float = 0.0


@dataclass
class WorkCurve:  # analysis.hpp:23-26
    layer: int = 0
    points: list[WorkCurvePoint] = field(default_factory=list)


@dataclass
class ConcavityEntry:  # analysis.hpp:35-40
    index: int = 0
    second_diff: float = 0.0
    threshold: float = 0.0
    violation: bool = False


@dataclass
class ConcavityReport:  # analysis.hpp:42-45
    entries: list[ConcavityEntry] = field(default_factory=list)
    passed: bool = True


def draw_seeds(num_vertices: int, batch_size: int, seed: int, tag: int) -> np.ndarray:
    """analysis.cpp:15-31: batch_size distinct vertices, deterministic in (seed, tag)."""
    if batch_size > num_vertices:
        raise InputError("seed draw: batch size exceeds vertex count")
    return first_distinct(hash_bits(seed, [8, tag]), num_vertices, batch_size).astype(np.uint32)


def draw_edges(indptr: np.ndarray, indices: np.ndarray, batch_size: int, seed: int,
               tag: int) -> np.ndarray:
    """analysis.cpp:34-54: batch_size distinct edge slots as (src, dst) pairs."""
    m = len(indices)
    if batch_size > m:
        raise InputError("seed draw: batch size exceeds edge count")
    e = first_distinct(hash_bits(seed, [8, tag, 1]), m, batch_size).astype(np.int64)
    dst = np.searchsorted(indptr, e.astype(np.uint64), side="right") - 1
    return np.stack([indices[e], dst.astype(np.uint32)], axis=1).astype(np.uint32)


def _mean_se(xs: list[float]) -> tuple[float, float]:
    """analysis.cpp:61-74, summed in trial order."""
    if not xs:
        return 0.0, 0.0
    s = 0.0
    for x in xs:
        s += x
    mean = s / len(xs)
    if len(xs) < 2:
        return mean, 0.0
    ss = 0.0
    for x in xs:
        ss += (x - mean) * (x - mean)
    return mean, math.sqrt(ss / (len(xs) - 1) / len(xs))


def work_curve(g: Graph, cfg: SamplerConfig, batch_sizes, trials: int, num_layers: int,
               seed: int, mode: SeedMode = SeedMode.kNode,
               trials_per_launch: int = 8) -> WorkCurve:
    """analysis.cpp:78-124 on the GPU: mean and standard error of |S^L| over
    `trials` batches per batch size."""
    if trials == 0:
        raise InputError("work_curve: trials must be >= 1")
    sizes = [int(b) for b in batch_sizes]
    curve = WorkCurve(layer=num_layers)
    csr = g.download() if mode == SeedMode.kEdge else None
    seeds: list[list[np.ndarray]] = []
    for bi, b in enumerate(sizes):
        if bi > 0 and b <= sizes[bi - 1]:
            raise InputError("work_curve: batch sizes must be strictly increasing")
        row = []
        for t in range(trials):
            tag = hash_bits(seed, [b, t])
            if mode == SeedMode.kNode:
                row.append(draw_seeds(g.num_vertices, b, seed, tag))
            else:
                edges = draw_edges(csr[0], csr[1], b, seed, tag)
                row.append(edge_pred_seeds(csr[0], csr[1], edges, hash_bits(seed, [tag, 7]),
                                           g.num_vertices))
        seeds.append(row)
    # one plan for the whole curve: G trials per launch, sized for the largest
    G = max(1, min(trials, trials_per_launch))
    plan = Plan(g, None, num_layers, cfg, max(1, max(len(s) for r in seeds for s in r)),
                parts=G)
    empty, idle = np.zeros(0, np.uint32), SeedSchedule.plain(0)
    for b, row in zip(sizes, seeds):
        sl: list[float] = []
        for c0 in range(0, trials, G):
            cs = row[c0:c0 + G]
            cz = [SeedSchedule(1, z, z, 0)
                  for z in (hash_bits(seed, [hash_bits(seed, [b, t]), 9])
                            for t in range(c0, c0 + len(cs)))]
            n = len(cs)
            plan.sample_multi(cs + [empty] * (G - n), cz + [idle] * (G - n))
            meta = plan.all_layer_sizes()
            sl += [float(meta[p, num_layers - 1, 4]) for p in range(n)]
        mean, se = _mean_se(sl)
        curve.points.append(WorkCurvePoint(b, mean, se, mean / b, se / b))
    return curve


def concavity_check(curve: WorkCurve) -> ConcavityReport:
    """analysis.cpp:126-151: every divided second difference of mean |S^L|
    must stay below +2 pooled standard errors."""
    pts = curve.points
    if len(pts) < 3:
        raise InputError("concavity_check: need at least 3 batch sizes")
    rep = ConcavityReport()
    for i in range(1, len(pts) - 1):
        h0 = float(pts[i].batch_size - pts[i - 1].batch_size)
        h1 = float(pts[i + 1].batch_size - pts[i].batch_size)
        slope0 = (pts[i].mean_sl - pts[i - 1].mean_sl) / h0
        slope1 = (pts[i + 1].mean_sl - pts[i].mean_sl) / h1
        var = (pts[i - 1].se_sl * pts[i - 1].se_sl / (h0 * h0)
               + pts[i + 1].se_sl * pts[i + 1].se_sl / (h1 * h1)
               + pts[i].se_sl * pts[i].se_sl * (1.0 / h0 + 1.0 / h1) * (1.0 / h0 + 1.0 / h1))
        e = ConcavityEntry(i, slope1 - slope0, 2.0 * math.sqrt(var))
        e.violation = e.second_diff > e.threshold
        if e.violation:
            rep.passed = False
        rep.entries.append(e)
    return rep
