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


def draw_from_pool(pool: np.ndarray, count: int, seed: int, tag: int) -> np.ndarray:
    pool = np.asarray(pool, dtype=np.uint32)
    n = len(pool)
    if count > n:
        raise ValueError("not enough vertices in pool to draw batch")
    pfx = hash_bits(seed, [8, tag])
    used = np.zeros(n, dtype=bool)
    out = np.empty(count, dtype=np.uint32)
    got, attempt = 0, 0
    while got < count:
        chunk = max(2 * (count - got), 64)
        att = np.arange(attempt, attempt + chunk, dtype=np.uint64)
        h = _mix64(_M(pfx) ^ att)
        u = (h >> _M(11)).astype(np.float64) * 2.0 ** -53
        idx = np.minimum((u * float(n)).astype(np.uint64), n - 1).astype(np.int64)
        for i in idx:  # sequential rejection of repeats, in attempt order
            if not used[i]:
                used[i] = True
                out[got] = pool[i]
                got += 1
                if got == count:
                    break
        attempt += chunk
    return out


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
