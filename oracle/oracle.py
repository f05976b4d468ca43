"""TEST INFRASTRUCTURE ONLY — the CPU checker, never the product path.

ctypes front-end over the two CPU checkers built by ``oracle/Makefile``:

* ``impl="restated"`` — ``oracle/liboracle.so``, the plain-C restatement of the
  reference algorithm (coopbatch_oracle.c; every function cites the reference
  file:line it restates);
* ``impl="reference"`` — ``oracle/_ref/libcoopbatch_ref.so``, the reference's own
  C++ sources (/root/reference/proj/src) compiled unmodified, behind the
  ``ref_capi.cpp`` shim.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs import
this module. Results use the same plain-dict layout as the product's
``paper_2310_12403_b200.coopbatch`` so parity checks are ``np.array_equal``.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OB_PATH = os.path.join(HERE, "liboracle.so")
RF_PATH = os.path.join(HERE, "_ref", "libcoopbatch_ref.so")

KAPPA_INF = (1 << 64) - 1
FULL, NS, LABOR0 = 0, 1, 2


class OracleError(ValueError):
    """The checker rejected its input (reference coopbatch::InputError)."""


class Sched(C.Structure):
    _fields_ = [("kappa", C.c_uint64), ("z1", C.c_uint64), ("z2", C.c_uint64),
                ("iteration", C.c_uint64)]


class Block(C.Structure):
    _fields_ = [("layer", C.c_int32), ("n_dst", C.c_uint64), ("n_src", C.c_uint64),
                ("n_edges", C.c_uint64), ("dst", C.POINTER(C.c_uint32)),
                ("src", C.POINTER(C.c_uint32)), ("edges", C.POINTER(C.c_uint32)),
                ("dst_pos", C.POINTER(C.c_uint32))]


class Stack(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("blocks", C.POINTER(Block))]


class Exchange(C.Structure):
    _fields_ = [("layer", C.c_int32), ("num_parts", C.c_uint32),
                ("send_counts", C.POINTER(C.c_uint64)),
                ("owner_row_counts", C.POINTER(C.c_uint64)),
                ("loc_len", C.POINTER(C.c_uint64)),
                ("loc_part", C.POINTER(C.POINTER(C.c_uint32))),
                ("loc_row", C.POINTER(C.POINTER(C.c_uint64)))]


class Coop(C.Structure):
    _fields_ = [("num_parts", C.c_uint32), ("num_layers", C.c_int32),
                ("stacks", C.POINTER(Stack)), ("exchanges", C.POINTER(Exchange)),
                ("owner_len", C.POINTER(C.c_uint64)),
                ("owner_sets", C.POINTER(C.POINTER(C.c_uint32)))]


_P = C.c_void_p
_u64, _u32, _i32, _f64 = C.c_uint64, C.c_uint32, C.c_int32, C.c_double

_libs: dict[str, C.CDLL] = {}


def available(impl: str = "restated") -> bool:
    return os.path.exists(OB_PATH if impl == "restated" else RF_PATH)


def lib(impl: str = "restated") -> C.CDLL:
    if impl in _libs:
        return _libs[impl]
    path = OB_PATH if impl == "restated" else RF_PATH
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not built (run __graft_entry__.build())")
    L = C.CDLL(path)
    pre = "ob_" if impl == "restated" else "rf_"
    L.last_error = getattr(L, pre + "last_error")
    L.last_error.restype = C.c_char_p
    _libs[impl] = L
    if impl == "restated":
        L.ob_mix64.restype = _u64
        L.ob_mix64.argtypes = [_u64]
        L.ob_hash_bits.restype = _u64
        L.ob_hash_bits.argtypes = [_u64, _P, C.c_int]
        L.ob_hash_uniform.restype = _f64
        L.ob_hash_uniform.argtypes = [_u64, _P, C.c_int]
        L.ob_phi.restype = _f64
        L.ob_phi.argtypes = [_f64]
        L.ob_inverse_phi.restype = _f64
        L.ob_inverse_phi.argtypes = [_f64]
        L.ob_normal_from_bits.restype = _f64
        L.ob_normal_from_bits.argtypes = [_u64]
        L.ob_labor_variate.restype = _f64
        L.ob_labor_variate.argtypes = [C.POINTER(Sched), C.c_int, _u32]
        L.ob_sched_make.argtypes = [_u64, _u64, C.POINTER(Sched)]
        L.ob_sched_advance.argtypes = [C.POINTER(Sched)]
        L.ob_rmat.argtypes = [_u64, _u64, _u64, C.POINTER(C.POINTER(_u64)),
                              C.POINTER(C.POINTER(_u32))]
        L.ob_rmat_par.argtypes = L.ob_rmat.argtypes
        L.ob_build_csr.argtypes = [_P, _P, _u64, _u64, _P, _P]
        L.ob_partition_random.argtypes = [_u64, _u32, _u64, _P]
        L.ob_sample_block.argtypes = [_P, _P, _u64, _P, _u64, C.c_int, _u32,
                                      C.POINTER(Sched), C.c_int, C.POINTER(Block)]
        L.ob_expand.argtypes = [_P, _P, _u64, _P, _u64, C.c_int, C.c_int, _P,
                                C.POINTER(Sched), C.POINTER(Stack)]
        L.ob_coop_sample.argtypes = [_P, _P, _u64, _P, _u32, _P, _P, C.c_int, C.c_int,
                                     _P, C.POINTER(Sched), C.POINTER(Coop)]
        L.ob_block_free.argtypes = [C.POINTER(Block)]
        L.ob_stack_free.argtypes = [C.POINTER(Stack)]
        L.ob_coop_free.argtypes = [C.POINTER(Coop)]
        L.ob_feature_rows.argtypes = [_u64, _u32, C.c_int, _P, _u64, _P]
        L.ob_lru_new.restype = _P
        L.ob_lru_new.argtypes = [_u64]
        L.ob_lru_access.argtypes = [_P, _u32]
        L.ob_lru_free.argtypes = [_P]
        L.ob_access_order.argtypes = [_P, _u64, _u64, _P]
        L.ob_stack_fingerprint.restype = _u64
        L.ob_stack_fingerprint.argtypes = [C.POINTER(Stack)]
        L.ob_draw_from_pool.argtypes = [_P, _u64, _u64, _u64, _u64, _P]
        L.ob_free.argtypes = [_P]
    else:
        L.rf_mix64.restype = _u64
        L.rf_mix64.argtypes = [_u64]
        L.rf_hash_bits.restype = _u64
        L.rf_hash_bits.argtypes = [_u64, _P, C.c_int]
        L.rf_phi.restype = _f64
        L.rf_phi.argtypes = [_f64]
        L.rf_inverse_phi.restype = _f64
        L.rf_inverse_phi.argtypes = [_f64]
        L.rf_normal_from_bits.restype = _f64
        L.rf_normal_from_bits.argtypes = [_u64]
        L.rf_labor_variate.restype = _f64
        L.rf_labor_variate.argtypes = [C.POINTER(Sched), C.c_int, _u32]
        L.rf_sched_make.argtypes = [_u64, _u64, C.POINTER(Sched)]
        L.rf_sched_advance.argtypes = [C.POINTER(Sched)]
        L.rf_graph_new.restype = _P
        L.rf_graph_new.argtypes = [_P, _P, _u64, _u64]
        L.rf_graph_free.argtypes = [_P]
        L.rf_graph_set_weights.argtypes = [_P, _P, _u64]
        L.rf_validate_csr.argtypes = [_P]
        L.rf_generate_powerlaw.argtypes = [_u64, _f64, _f64, _u64,
                                           C.POINTER(C.POINTER(_u64)),
                                           C.POINTER(C.POINTER(_u32)), C.POINTER(_u64)]
        L.rf_build_csr.argtypes = [_P, _P, _u64, _u64, _P, _P]
        L.rf_partition_random.argtypes = [_u64, _u32, _u64, _P]
        L.rf_sample_block.argtypes = [_P, _P, _u64, C.c_int, _u32, C.POINTER(Sched),
                                      C.c_int, C.POINTER(Block)]
        L.rf_sample_labor0.argtypes = [_P, _P, _u64, _u32, _P, C.c_int, C.POINTER(Block)]
        L.rf_expand.argtypes = [_P, _P, _u64, C.c_int, C.c_int, _P, C.POINTER(Sched),
                                C.POINTER(Stack)]
        L.rf_coop_sample.argtypes = [_P, _P, _u32, _P, _P, C.c_int, C.c_int, _u32,
                                     C.POINTER(Sched), C.POINTER(Coop)]
        L.rf_block_free.argtypes = [C.POINTER(Block)]
        L.rf_stack_free.argtypes = [C.POINTER(Stack)]
        L.rf_coop_free.argtypes = [C.POINTER(Coop)]
        L.rf_free.argtypes = [_P]
        L.rf_features_new.restype = _P
        L.rf_features_new.argtypes = [_u64, _u32, _u32, _u64]
        L.rf_features_free.argtypes = [_P]
        L.rf_load_rows.argtypes = [_P, _P, _u64, _P]
        L.rf_all_to_all_forward.argtypes = [C.POINTER(Coop), C.c_int, _P, _P, _u32, _P]
        L.rf_step.argtypes = [_P, _P, C.c_int, _P, _u32, _P, _P, C.c_int, C.c_int, _u32,
                              C.POINTER(Sched), C.POINTER(_f64), C.POINTER(_f64),
                              C.POINTER(_u64)]
        L.rf_step_onfly.argtypes = [_P, _u64, _u32, C.c_int, _P, _u32, _P, _P, C.c_int,
                                    C.c_int, _u32, C.POINTER(Sched), _P, _P, _P]
        L.rf_train_step.argtypes = [_P, _P, C.c_int, _P, _u32, _P, _P, C.c_int, C.c_int, _u32,
                                    C.POINTER(Sched), _u32, _u64, C.POINTER(_f64), _P]
        L.rf_cross_edge_ratio.argtypes = [_P, _P, _u32, C.POINTER(_f64)]
        L.rf_edge_pred_seeds.argtypes = [_P, _P, _u64, _u64, _P, C.POINTER(_u64)]
        L.rf_work_curve.argtypes = [_P, C.c_int, _u32, _P, _u64, _u32, C.c_int, _u64,
                                    C.c_int, _P]
        L.rf_concavity_check.argtypes = [_P, _P, _P, _u64, _P, _P, _P, C.POINTER(C.c_int)]
        L.rf_save_csr.argtypes = [_P, C.c_char_p]
        L.rf_load_csr.argtypes = [C.c_char_p, C.POINTER(_u64), C.POINTER(_u64),
                                  C.POINTER(C.POINTER(_u64)), C.POINTER(C.POINTER(_u32))]
        L.rf_lru_new.restype = _P
        L.rf_lru_new.argtypes = [_u64]
        L.rf_lru_access.argtypes = [_P, _u32]
        L.rf_lru_free.argtypes = [_P]
        L.rf_dependent_experiment.argtypes = [_P, C.c_int, _u64, _u64, _u64, _u64,
                                              C.c_int, _u32, C.c_int, _u32, _u32, _u64,
                                              _P, _P, _P, C.POINTER(_f64)]
    return L


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _check(rc: int, L: C.CDLL):
    if rc != 0:
        raise OracleError(L.last_error().decode())


def _arr(p, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(p, shape=(int(n),)).astype(dtype, copy=True)


def _block(b: Block) -> dict:
    return {
        "layer": int(b.layer),
        "dst": _arr(b.dst, b.n_dst, np.uint32),
        "src": _arr(b.src, b.n_src, np.uint32),
        "edges": _arr(b.edges, 2 * b.n_edges, np.uint32).reshape(-1, 2),
        "dst_pos": _arr(b.dst_pos, b.n_dst, np.uint32),
    }


def _stack(s: Stack) -> list[dict]:
    return [_block(s.blocks[l]) for l in range(s.num_layers)]


# --------------------------------------------------------------------- rng ---

def make_sched(kappa: int, root_seed: int, impl: str = "restated") -> Sched:
    s = Sched()
    getattr(lib(impl), "ob_sched_make" if impl == "restated" else "rf_sched_make")(
        kappa, root_seed, C.byref(s))
    return s


def plain_sched(seed: int) -> Sched:
    """test_samplers.cpp:45-50 plain_schedule: kappa 1, z1 = z2 = seed."""
    return Sched(1, seed, seed, 0)


def advance(s: Sched, impl: str = "restated") -> Sched:
    t = Sched(s.kappa, s.z1, s.z2, s.iteration)
    getattr(lib(impl), "ob_sched_advance" if impl == "restated" else "rf_sched_advance")(
        C.byref(t))
    return t


def hash_bits(seed: int, ids, impl: str = "restated") -> int:
    a = np.asarray(ids, dtype=np.uint64)
    L = lib(impl)
    f = L.ob_hash_bits if impl == "restated" else L.rf_hash_bits
    return int(f(seed, _ptr(a), len(a)))


# ------------------------------------------------------------------- graph ---

@dataclass
class CSR:
    indptr: np.ndarray   # u64[n+1]
    indices: np.ndarray  # u32[m]
    weights: np.ndarray | None = None  # f32[m] (graph.hpp:25), reference-only

    @property
    def n(self) -> int:
        return len(self.indptr) - 1

    @property
    def m(self) -> int:
        return len(self.indices)


def rmat(n: int, m: int, seed: int, parallel: bool | None = None) -> CSR:
    """Hash-keyed R-MAT. `parallel` (default: m > 2^22) uses the bucketed
    multi-threaded form, which builds the same CSR."""
    L = lib("restated")
    ip = C.POINTER(_u64)()
    ix = C.POINTER(_u32)()
    if parallel is None:
        parallel = m > (1 << 22)
    fn = L.ob_rmat_par if parallel else L.ob_rmat
    _check(fn(n, m, seed, C.byref(ip), C.byref(ix)), L)
    g = CSR(_arr(ip, n + 1, np.uint64), _arr(ix, m, np.uint32))
    L.ob_free(C.cast(ip, C.c_void_p))
    L.ob_free(C.cast(ix, C.c_void_p))
    return g


def generate_powerlaw(n: int, deg: float, skew: float, seed: int) -> CSR:
    """The reference's own generator (graph.cpp:111-151), for fixtures."""
    L = lib("reference")
    ip = C.POINTER(_u64)()
    ix = C.POINTER(_u32)()
    m = _u64()
    _check(L.rf_generate_powerlaw(n, deg, skew, seed, C.byref(ip), C.byref(ix),
                                  C.byref(m)), L)
    g = CSR(_arr(ip, n + 1, np.uint64), _arr(ix, m.value, np.uint32))
    L.rf_free(C.cast(ip, C.c_void_p))
    L.rf_free(C.cast(ix, C.c_void_p))
    return g


def build_csr(src, dst, n: int, impl: str = "restated") -> CSR:
    src = np.ascontiguousarray(src, dtype=np.uint32)
    dst = np.ascontiguousarray(dst, dtype=np.uint32)
    ip = np.zeros(n + 1, dtype=np.uint64)
    ix = np.zeros(len(src), dtype=np.uint32)
    L = lib(impl)
    f = L.ob_build_csr if impl == "restated" else L.rf_build_csr
    _check(f(_ptr(src), _ptr(dst), len(src), n, _ptr(ip), _ptr(ix)), L)
    return CSR(ip, ix)


class RefGraph:
    """A coopbatch::Graph inside the compiled reference."""

    def __init__(self, g: CSR):
        self.csr = g
        self.L = lib("reference")
        self.h = self.L.rf_graph_new(_ptr(g.indptr), _ptr(g.indices), g.n, g.m)
        if getattr(g, "weights", None) is not None:
            w = np.ascontiguousarray(g.weights, dtype=np.float32)
            self.L.rf_graph_set_weights(self.h, _ptr(w), len(w))

    def __del__(self):
        if getattr(self, "h", None):
            self.L.rf_graph_free(self.h)
            self.h = None


def train_step_reference(g: CSR, mode: int, owner, parts: int, per_pe_seeds, L: int, kind: int,
                         fanout: int, sched: Sched, dim: int, classes: int, feat_seed: int,
                         hidden: int, model_seed: int, grad_sizes):
    """The compiled reference's coop_train_step (mode 0) / indep_train_step
    (mode 1) with FeatureStore::synth(n, dim, classes, feat_seed) and
    GcnModel::init(dim, hidden, classes, L, model_seed)."""
    rg = RefGraph(g)
    fs = RefFeatureStore(g.n, dim, feat_seed, classes)
    flat = np.ascontiguousarray(np.concatenate([np.asarray(s, np.uint32) for s in per_pe_seeds]),
                                dtype=np.uint32)
    off = np.zeros(parts + 1, np.uint64)
    off[1:] = np.cumsum([len(s) for s in per_pe_seeds])
    own = None if owner is None else np.ascontiguousarray(owner, dtype=np.uint32)
    gw = np.zeros(int(sum(grad_sizes)), np.float64)
    loss = C.c_double()
    _check(rg.L.rf_train_step(rg.h, fs.h, mode, _ptr(own), parts, _ptr(flat), _ptr(off), L, kind,
                              fanout, C.byref(sched), hidden, model_seed, C.byref(loss),
                              _ptr(gw)), rg.L)
    return loss.value, gw


def cross_edge_ratio_reference(g: CSR, owner: np.ndarray, parts: int) -> float:
    rg = RefGraph(g)
    out = C.c_double()
    own = np.ascontiguousarray(owner, dtype=np.uint32)
    _check(rg.L.rf_cross_edge_ratio(rg.h, _ptr(own), parts, C.byref(out)), rg.L)
    return out.value


def edge_pred_seeds_reference(g: CSR, edges, epoch_seed: int) -> np.ndarray:
    """The reference's edge_pred_seeds (samplers.cpp:356-393)."""
    rg = RefGraph(g)
    uv = np.ascontiguousarray(edges, dtype=np.uint32).reshape(-1, 2)
    out = np.zeros(3 * len(uv) + 1, np.uint32)
    n = C.c_uint64()
    _check(rg.L.rf_edge_pred_seeds(rg.h, _ptr(uv), len(uv), epoch_seed, _ptr(out),
                                   C.byref(n)), rg.L)
    return out[: n.value]


def sample_labor0_reference(g: CSR, seeds, k: int, table, layer: int = 0) -> dict:
    """The reference's sample_labor0 (samplers.cpp:305-312) with r(t) = table[t]."""
    rg = RefGraph(g)
    sd = np.ascontiguousarray(seeds, dtype=np.uint32)
    tb = np.ascontiguousarray(table, dtype=np.float64)
    b = Block()
    _check(rg.L.rf_sample_labor0(rg.h, _ptr(sd), len(sd), k, _ptr(tb), layer, C.byref(b)), rg.L)
    out = _block(b)
    rg.L.rf_block_free(C.byref(b))
    return out


def work_curve_reference(g: CSR, kind: int, fanout: int, sizes, trials: int, num_layers: int,
                         seed: int, edge_mode: bool = False) -> np.ndarray:
    """The reference's work_curve (analysis.cpp:78-124): rows of (mean_sl,
    se_sl, work_per_seed, se_work) per batch size."""
    rg = RefGraph(g)
    sz = np.ascontiguousarray(sizes, dtype=np.uint64)
    out = np.zeros((len(sz), 4), np.float64)
    _check(rg.L.rf_work_curve(rg.h, kind, fanout, _ptr(sz), len(sz), trials, num_layers, seed,
                              int(edge_mode), _ptr(out)), rg.L)
    return out


def concavity_check_reference(sizes, mean, se):
    """The reference's concavity_check (analysis.cpp:126-151): (second_diff,
    threshold, violation) per interior point and the overall pass flag."""
    L = lib("reference")
    sz = np.ascontiguousarray(sizes, dtype=np.uint64)
    mu = np.ascontiguousarray(mean, dtype=np.float64)
    sd = np.ascontiguousarray(se, dtype=np.float64)
    n = len(sz)
    d2, thr = np.zeros(max(n - 2, 1)), np.zeros(max(n - 2, 1))
    vio = np.zeros(max(n - 2, 1), np.int32)
    ok = C.c_int()
    _check(L.rf_concavity_check(_ptr(sz), _ptr(mu), _ptr(sd), n, _ptr(d2), _ptr(thr), _ptr(vio),
                                C.byref(ok)), L)
    return d2[: n - 2], thr[: n - 2], vio[: n - 2].astype(bool), bool(ok.value)


def save_csr_reference(g: CSR, path: str):
    """The reference's save_csr (graph.cpp:216-229) on this CSR."""
    rg = RefGraph(g)
    _check(rg.L.rf_save_csr(rg.h, str(path).encode()), rg.L)


def load_csr_reference(path: str) -> CSR:
    """The reference's load_csr (graph.cpp:231-252), incl. validate_csr."""
    L = lib("reference")
    n, m = C.c_uint64(), C.c_uint64()
    ip, ix = C.POINTER(_u64)(), C.POINTER(_u32)()
    _check(L.rf_load_csr(str(path).encode(), C.byref(n), C.byref(m), C.byref(ip), C.byref(ix)), L)
    indptr = np.ctypeslib.as_array(ip, (n.value + 1,)).copy()
    indices = np.ctypeslib.as_array(ix, (max(m.value, 1),))[: m.value].copy()
    L.rf_free(C.cast(ip, _P))
    L.rf_free(C.cast(ix, _P))
    return CSR(indptr, indices)


def partition_random(n: int, parts: int, seed: int, impl: str = "restated") -> np.ndarray:
    owner = np.zeros(n, dtype=np.uint32)
    L = lib(impl)
    f = L.ob_partition_random if impl == "restated" else L.rf_partition_random
    _check(f(n, parts, seed, _ptr(owner)), L)
    return owner


def part_members(owner: np.ndarray, parts: int) -> list[np.ndarray]:
    """partition.cpp:99-105: vertices of each part, ascending."""
    return [np.flatnonzero(owner == p).astype(np.uint32) for p in range(parts)]


# ---------------------------------------------------------------- sampling ---

def _fanouts(fanout, L: int) -> np.ndarray:
    if np.isscalar(fanout):
        return np.full(L, int(fanout), dtype=np.uint32)
    f = np.asarray(fanout, dtype=np.uint32)
    assert len(f) == L
    return f


def sample_block(g, seeds, kind: int, fanout: int, sched: Sched, layer: int,
                 impl: str = "restated") -> dict:
    seeds = np.ascontiguousarray(seeds, dtype=np.uint32)
    b = Block()
    if impl == "restated":
        L = lib(impl)
        _check(L.ob_sample_block(_ptr(g.indptr), _ptr(g.indices), g.n, _ptr(seeds),
                                 len(seeds), kind, fanout, C.byref(sched), layer,
                                 C.byref(b)), L)
        out = _block(b)
        L.ob_block_free(C.byref(b))
    else:
        rg = g if isinstance(g, RefGraph) else RefGraph(g)
        L = rg.L
        _check(L.rf_sample_block(rg.h, _ptr(seeds), len(seeds), kind, fanout,
                                 C.byref(sched), layer, C.byref(b)), L)
        out = _block(b)
        L.rf_block_free(C.byref(b))
    return out


def expand(g, seeds, num_layers: int, kind: int, fanout, sched: Sched,
           impl: str = "restated") -> list[dict]:
    seeds = np.ascontiguousarray(seeds, dtype=np.uint32)
    fo = _fanouts(fanout, num_layers)
    s = Stack()
    if impl == "restated":
        L = lib(impl)
        _check(L.ob_expand(_ptr(g.indptr), _ptr(g.indices), g.n, _ptr(seeds), len(seeds),
                           num_layers, kind, _ptr(fo), C.byref(sched), C.byref(s)), L)
        out = _stack(s)
        L.ob_stack_free(C.byref(s))
    else:
        rg = g if isinstance(g, RefGraph) else RefGraph(g)
        L = rg.L
        _check(L.rf_expand(rg.h, _ptr(seeds), len(seeds), num_layers, kind, _ptr(fo),
                           C.byref(sched), C.byref(s)), L)
        out = _stack(s)
        L.rf_stack_free(C.byref(s))
    return out


def _coop_dict(c: Coop) -> dict:
    P, Lh = c.num_parts, c.num_layers
    ex = []
    for l in range(Lh):
        e = c.exchanges[l]
        ex.append({
            "layer": int(e.layer),
            "send_counts": _arr(e.send_counts, P * P, np.uint64).reshape(P, P),
            "owner_row_counts": _arr(e.owner_row_counts, P, np.uint64),
            "loc_part": [_arr(e.loc_part[p], e.loc_len[p], np.uint32) for p in range(P)],
            "loc_row": [_arr(e.loc_row[p], e.loc_len[p], np.uint64) for p in range(P)],
        })
    return {
        "stacks": [_stack(c.stacks[p]) for p in range(P)],
        "exchanges": ex,
        "owner_sets": [_arr(c.owner_sets[p], c.owner_len[p], np.uint32) for p in range(P)],
    }


def coop_sample(g, owner, parts: int, per_pe_seeds, num_layers: int, kind: int,
                fanout, sched: Sched, impl: str = "restated", keep_handle=False):
    owner = np.ascontiguousarray(owner, dtype=np.uint32)
    flat = np.ascontiguousarray(np.concatenate(
        [np.asarray(s, dtype=np.uint32) for s in per_pe_seeds]) if per_pe_seeds
        else np.zeros(0, np.uint32), dtype=np.uint32)
    off = np.zeros(len(per_pe_seeds) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(s) for s in per_pe_seeds])
    fo = _fanouts(fanout, num_layers)
    c = Coop()
    if impl == "restated":
        L = lib(impl)
        if len(per_pe_seeds) != parts:
            raise OracleError("coop_sample: seed lists must match the partition count")
        _check(L.ob_coop_sample(_ptr(g.indptr), _ptr(g.indices), g.n, _ptr(owner), parts,
                                _ptr(flat), _ptr(off), num_layers, kind, _ptr(fo),
                                C.byref(sched), C.byref(c)), L)
        out = _coop_dict(c)
        L.ob_coop_free(C.byref(c))
        return out
    rg = g if isinstance(g, RefGraph) else RefGraph(g)
    L = rg.L
    if len(per_pe_seeds) != parts:
        raise OracleError("coop_sample: seed lists must match the partition count")
    if len(set(fo.tolist())) > 1:
        raise OracleError("reference coop_sample has a single fanout")
    _check(L.rf_coop_sample(rg.h, _ptr(owner), parts, _ptr(flat), _ptr(off), num_layers,
                            kind, int(fo[0]) if len(fo) else 1, C.byref(sched),
                            C.byref(c)), L)
    out = _coop_dict(c)
    if keep_handle:
        return out, c
    L.rf_coop_free(C.byref(c))
    return out


def coop_free_reference(c: Coop):
    lib("reference").rf_coop_free(C.byref(c))


# ---------------------------------------------------------------- features ---

DTYPES = {"f64": (0, np.float64), "f32": (1, np.float32), "f16": (2, np.float16)}


def feature_rows(seed: int, dim: int, dtype: str, ids) -> np.ndarray:
    """coop.cpp:369-371 values for `ids`, rounded once to `dtype`."""
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    code, npdt = DTYPES[dtype]
    out = np.zeros((len(ids), dim), dtype=npdt)
    lib("restated").ob_feature_rows(seed, dim, code, _ptr(ids), len(ids), _ptr(out))
    return out


class RefFeatureStore:
    """coopbatch::FeatureStore::synth (coop.cpp:359-376), f64 table."""

    def __init__(self, n: int, dim: int, seed: int, classes: int = 2):
        self.L = lib("reference")
        self.dim = dim
        self.h = self.L.rf_features_new(n, dim, classes, seed)

    def load_rows(self, ids) -> np.ndarray:
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        out = np.zeros((len(ids), self.dim), dtype=np.float64)
        self.L.rf_load_rows(self.h, _ptr(ids), len(ids), _ptr(out))
        return out

    def __del__(self):
        if getattr(self, "h", None):
            self.L.rf_features_free(self.h)
            self.h = None


# ------------------------------------------------------------------- cache ---

class Lru:
    def __init__(self, cap: int, impl: str = "restated"):
        self.L = lib(impl)
        self.impl = impl
        self.h = (self.L.ob_lru_new if impl == "restated" else self.L.rf_lru_new)(cap)
        if not self.h:
            raise OracleError("LruCache: capacity must be >= 1")

    def access(self, key: int) -> bool:
        """True on miss."""
        f = self.L.ob_lru_access if self.impl == "restated" else self.L.rf_lru_access
        return bool(f(self.h, key))

    def __del__(self):
        if getattr(self, "h", None):
            (self.L.ob_lru_free if self.impl == "restated" else self.L.rf_lru_free)(self.h)
            self.h = None


def access_order(ids, key: int) -> np.ndarray:
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    out = np.zeros_like(ids)
    lib("restated").ob_access_order(_ptr(ids), len(ids), key, _ptr(out))
    return out


def stack_fingerprint(stack: list[dict]) -> int:
    """cache.cpp:123-133 over a dict-form stack (pure numpy restatement)."""
    L = lib("restated")
    blocks = (Block * len(stack))()
    keep = []
    for i, b in enumerate(stack):
        arrs = [np.ascontiguousarray(b[k], dtype=np.uint32)
                for k in ("dst", "src", "edges", "dst_pos")]
        keep.append(arrs)
        blocks[i].layer = b["layer"]
        blocks[i].n_dst = len(arrs[0])
        blocks[i].n_src = len(arrs[1])
        blocks[i].n_edges = arrs[2].size // 2
        blocks[i].dst = arrs[0].ctypes.data_as(C.POINTER(C.c_uint32))
        blocks[i].src = arrs[1].ctypes.data_as(C.POINTER(C.c_uint32))
        blocks[i].edges = arrs[2].ctypes.data_as(C.POINTER(C.c_uint32))
        blocks[i].dst_pos = arrs[3].ctypes.data_as(C.POINTER(C.c_uint32))
    s = Stack(len(stack), C.cast(blocks, C.POINTER(Block)))
    return int(L.ob_stack_fingerprint(C.byref(s)))


def draw_from_pool(pool, count: int, seed: int, tag: int) -> np.ndarray:
    pool = np.ascontiguousarray(pool, dtype=np.uint32)
    out = np.zeros(count, dtype=np.uint32)
    L = lib("restated")
    _check(L.ob_draw_from_pool(_ptr(pool), len(pool), count, seed, tag, _ptr(out)), L)
    return out


def draw_coop_seeds(owner: np.ndarray, parts: int, b: int, seed: int,
                    step: int) -> list[np.ndarray]:
    """cli.cpp:210-214: per-PE seeds draw_from_pool(members[p], b, seed,
    hash_bits(step, {p}))."""
    members = part_members(owner, parts)
    return [draw_from_pool(members[p], b, seed, hash_bits(step, [p])) for p in range(parts)]


def dependent_experiment(g, mode: int, kappa: int, batch: int, steps: int, capacity: int,
                         kind: int, fanout: int, L: int, dim: int, bps: int, seed: int):
    rg = g if isinstance(g, RefGraph) else RefGraph(g)
    fp = np.zeros(steps, np.uint64)
    sl = np.zeros(steps, np.uint64)
    by = np.zeros(steps, np.uint64)
    steady = C.c_double()
    _check(rg.L.rf_dependent_experiment(rg.h, mode, kappa, batch, steps, capacity, kind,
                                        fanout, L, dim, bps, seed, _ptr(fp), _ptr(sl),
                                        _ptr(by), C.byref(steady)), rg.L)
    return {"fingerprint": fp, "s_l": sl, "bytes": by, "steady": steady.value}


def reference_step(rg: RefGraph, fs: RefFeatureStore, mode: int, owner, parts: int,
                   per_pe_seeds, num_layers: int, kind: int, fanout: int, sched: Sched):
    """The reference's stock sample + load_rows (+ all_to_all_forward) path for
    one minibatch; returns (t_sample_s, t_gather_s, rows)."""
    flat = np.ascontiguousarray(np.concatenate(
        [np.asarray(s, dtype=np.uint32) for s in per_pe_seeds]), dtype=np.uint32)
    off = np.zeros(parts + 1, np.uint64)
    off[1:] = np.cumsum([len(s) for s in per_pe_seeds])
    own = None if owner is None else np.ascontiguousarray(owner, dtype=np.uint32)
    ts, tg, rows = C.c_double(), C.c_double(), C.c_uint64()
    _check(rg.L.rf_step(rg.h, fs.h, mode, _ptr(own), parts, _ptr(flat), _ptr(off), num_layers,
                        kind, fanout, C.byref(sched), C.byref(ts), C.byref(tg),
                        C.byref(rows)), rg.L)
    return ts.value, tg.value, rows.value


def reference_step_onfly(rg: RefGraph, feat_seed: int, dim: int, mode: int, owner,
                         parts: int, per_pe_seeds, num_layers: int, kind: int, fanout: int,
                         sched: Sched):
    """reference_step with load_rows replaced by rows computed from
    FeatureStore::synth's formula (for graphs whose f64 store does not fit);
    returns (t_sample_s, t_gather_s, rows)."""
    flat = np.ascontiguousarray(np.concatenate(
        [np.asarray(s, dtype=np.uint32) for s in per_pe_seeds]), dtype=np.uint32)
    off = np.zeros(parts + 1, np.uint64)
    off[1:] = np.cumsum([len(s) for s in per_pe_seeds])
    own = None if owner is None else np.ascontiguousarray(owner, dtype=np.uint32)
    ts, tg, rows = C.c_double(), C.c_double(), C.c_uint64()
    _check(rg.L.rf_step_onfly(rg.h, feat_seed, dim, mode, _ptr(own), parts, _ptr(flat),
                              _ptr(off), num_layers, kind, fanout, C.byref(sched),
                              C.byref(ts), C.byref(tg), C.byref(rows)), rg.L)
    return ts.value, tg.value, rows.value


def dependent_experiment_restated(g: CSR, kappa: int, batch: int, steps: int, capacity: int,
                                  kind: int, fanout: int, L: int, dim: int, bps: int,
                                  seed: int) -> dict:
    """run_dependent_experiment (cache.cpp:137-208), smoothed mode, composed from
    the restated pieces: Fisher-Yates order (hash(seed,{8,i})), SeedSchedule,
    expand, stack_fingerprint, access_order, LRU."""
    n = g.n
    b = min(batch, n)
    order = np.arange(n, dtype=np.uint32)
    for i in range(n, 1, -1):
        j = int(lib().ob_hash_uniform(seed, _ptr(np.array([8, i], np.uint64)), 2) * i)
        order[i - 1], order[min(j, i - 1)] = order[min(j, i - 1)], order[i - 1]
    spe = max(1, n // b)
    sched = make_sched(kappa, seed)
    lru = Lru(capacity)
    fp, sl, by = [], [], []
    for step in range(steps):
        slot = (step % spe) * b
        st = expand(g, order[slot:slot + b], L, kind, fanout, sched)
        sched = advance(sched)
        fp.append(stack_fingerprint(st))
        inputs = access_order(st[-1]["src"], hash_bits(seed, [step, 0xACCE55]))
        miss = sum(lru.access(int(v)) for v in inputs)
        sl.append(len(inputs))
        by.append(miss * dim * bps)
    return {"fingerprint": np.array(fp, np.uint64), "s_l": np.array(sl, np.uint64),
            "bytes": np.array(by, np.uint64)}
