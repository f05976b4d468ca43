"""Host-side minibatch seed draws, identical to the reference CLI's
``draw_from_pool`` (cli.cpp:121-139) and its per-PE tags (cli.cpp:210-214):
part p of step s draws b distinct vertices from its members with
``hash_uniform(seed, {kStreamSeedDraw=8, hash_bits(s, {p}), attempt})``.
Vectorised with numpy uint64 arithmetic (input generation, not the measured
path)."""
from __future__ import annotations

import numpy as np

from .coopbatch import hash_bits

_M = np.uint64


def _mix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + _M(0x9E3779B97F4A7C15)
        x = (x ^ (x >> _M(30))) * _M(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> _M(27))) * _M(0x94D049BB133111EB)
        return x ^ (x >> _M(31))


def first_distinct(prefix: int, space: int, count: int) -> np.ndarray:
    """The first `count` distinct values of the stream
    v_a = min(floor(U(mix64(prefix ^ a)) * space), space - 1), a = 0, 1, ...,
    in stream order: the rejection loops of draw_from_pool (cli.cpp:121-139),
    draw_seeds and draw_edges (analysis.cpp:15-54), vectorised."""
    if count == 0:
        return np.zeros(0, np.uint64)
    vals = np.zeros(0, np.uint64)
    attempt, chunk = 0, max(2 * count, 64)
    while True:
        att = np.arange(attempt, attempt + chunk, dtype=np.uint64)
        u = (_mix64(_M(prefix) ^ att) >> _M(11)).astype(np.float64) * 2.0 ** -53
        v = np.minimum((u * float(space)).astype(np.uint64), _M(space - 1))
        vals = np.concatenate([vals, v])
        attempt += chunk
        uniq, first = np.unique(vals, return_index=True)
        if len(uniq) >= count:
            first.sort()
            return vals[first[:count]]
        chunk *= 2


def draw_from_pool(pool: np.ndarray, count: int, seed: int, tag: int) -> np.ndarray:
    pool = np.asarray(pool, dtype=np.uint32)
    if count > len(pool):
        raise ValueError("not enough vertices in pool to draw batch")
    return pool[first_distinct(hash_bits(seed, [8, tag]), len(pool), count).astype(np.int64)]


def draw_batch(num_vertices: int, count: int, seed: int) -> np.ndarray:
    """acceptance.cpp:71-83: `count` distinct vertices from the stream
    hash_uniform(seed, {31337, attempt}) (the acceptance harness's global batch)."""
    return first_distinct(hash_bits(seed, [31337]), num_vertices, count).astype(np.uint32)


def split_by_owner(batch, owner: np.ndarray, parts: int) -> list[np.ndarray]:
    """acceptance.cpp:64-69: a global batch split into per-part seed lists by
    owner, batch order kept within a part."""
    b = np.asarray(batch, dtype=np.uint32)
    own = np.asarray(owner)[b]
    return [b[own == p] for p in range(parts)]


def coop_seeds(members: list[np.ndarray], b: int, seed: int, step: int) -> list[np.ndarray]:
    """Per-part seeds of one cooperative step (cli.cpp:210-214)."""
    return [draw_from_pool(members[p], b, seed, hash_bits(step, [p]))
            for p in range(len(members))]


def edge_pred_seeds(indptr: np.ndarray, indices: np.ndarray, edge_batch, epoch_seed: int,
                    num_vertices: int | None = None) -> np.ndarray:
    """samplers.cpp:356-393: seeds of an edge-prediction minibatch. For each
    (u, v): both endpoints (first occurrence order), then one negative endpoint
    w drawn uniformly with hash_uniform(seed, {kStreamEdgeNeg=6, u, v, attempt})
    that is neither the shared endpoint (u or v by the coin hash_uniform(seed,
    {kStreamEdgeCoin=5, u, v}) < 0.5) nor one of its in-neighbours; 100
    attempts, else InputError. Host-side input generation like
    draw_from_pool (the graph's CSR arrays come from Graph.download())."""
    from .coopbatch import InputError, hash_uniform
    n = len(indptr) - 1 if num_vertices is None else num_vertices
    out, seen = [], set()

    def push(x):
        if x not in seen:
            seen.add(x)
            out.append(x)
    for u, v in np.asarray(edge_batch, dtype=np.uint64).reshape(-1, 2):
        u, v = int(u), int(v)
        if u >= n or v >= n:
            raise InputError("vertex id out of range")
        push(u)
        push(v)
        shared = u if hash_uniform(epoch_seed, [5, u, v]) < 0.5 else v
        blocked = set(indices[indptr[shared]:indptr[shared + 1]].tolist())
        blocked.add(shared)
        for attempt in range(100):
            r = hash_uniform(epoch_seed, [6, u, v, attempt])
            w = min(int(r * float(n)), n - 1)
            if w in blocked:
                continue
            push(w)
            break
        else:
            raise InputError("edge_pred_seeds: no negative endpoint found for vertex "
                             f"{shared} after 100 attempts")
    return np.asarray(out, dtype=np.uint32)
