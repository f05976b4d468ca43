"""Loader for libcoopbatch_b200.so (the sm_100a kernels + C-ABI).

There is no fallback: if the shared library is missing, importing the product
API raises, so a GPU run can never silently degrade to a CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
# CB_LIB_PATH: an alternative in-tree build (A/B experiments under tools/)
LIB_PATH = os.environ.get("CB_LIB_PATH") or os.path.join(HERE, "libcoopbatch_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "coopbatch_cuda.h")


class Sched(C.Structure):
    _fields_ = [("kappa", C.c_uint64), ("z1", C.c_uint64), ("z2", C.c_uint64),
                ("iteration", C.c_uint64)]


_P = C.c_void_p
_u64, _u32 = C.c_uint64, C.c_uint32
_PP = C.POINTER(C.c_void_p)

_SIGS = {
    "cb_last_error": (C.c_char_p, []),
    "cb_version": (C.c_char_p, []),
    "cb_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "cb_graph_create_from_csr": (C.c_int, [_P, _P, _u64, _u64, C.c_int, _PP]),
    "cb_graph_generate_rmat": (C.c_int, [_u64, _u64, _u64, C.c_int, _PP]),
    "cb_graph_load_cbcs": (C.c_int, [C.c_char_p, C.c_int, _PP]),
    "cb_graph_set_weights": (C.c_int, [_P, _P]),
    "cb_plan_set_variate_source": (C.c_int, [_P, _P]),
    "cb_op_forward_rows": (C.c_int, [C.c_int, _u32, _P, _P, _P, _P, _u32, _P, _P]),
    "cb_op_reverse_rows": (C.c_int, [C.c_int, _u32, _P, _P, _P, _P, _u32, _P, C.c_int, _P]),
    "cb_op_gcn_block": (C.c_int, [C.c_int, _u64, _u64, _u64, _P, _P, _P, _u32, _P, _u32, C.c_int,
                                  _P, _P, _P, _P]),
    "cb_features_from_host": (C.c_int, [C.c_int, _u64, _u32, C.c_int, _P, _PP]),
    "cb_features_set_labels": (C.c_int, [_P, _P]),
    "cb_synth_host": (C.c_int, [C.c_int, _u64, _u32, _u32, _u64, _P, _P]),
    "cb_features_wrap_host": (C.c_int, [C.c_int, _u64, _u32, C.c_int, _P, _PP]),
    "cb_op_load_rows": (C.c_int, [_P, _P, _u64, _P]),
    "cb_gcn_model_create": (C.c_int, [C.c_int, C.c_int, _P, _P, C.c_int, _P, _PP]),
    "cb_graph_save_cbcs": (C.c_int, [_P, C.c_char_p]),
    "cb_graph_info": (C.c_int, [_P, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64)]),
    "cb_graph_download": (C.c_int, [_P, _P, _P]),
    "cb_graph_destroy": (None, [_P]),
    "cb_partition_random": (C.c_int, [_P, _u32, _u64, _PP]),
    "cb_partition_create": (C.c_int, [_P, _P, _u32, _PP]),
    "cb_partition_download": (C.c_int, [_P, _P]),
    "cb_partition_members": (C.c_int, [_P, _P, _P]),
    "cb_cross_edge_ratio": (C.c_int, [_P, _P, C.POINTER(_u64), C.POINTER(C.c_double)]),
    "cb_partition_destroy": (None, [_P]),
    "cb_features_synth": (C.c_int, [_P, _P, _u32, C.c_int, _u64, _PP]),
    "cb_features_info": (C.c_int, [_P, C.POINTER(_u32), C.POINTER(C.c_int), C.POINTER(_u64)]),
    "cb_features_destroy": (None, [_P]),
    "cb_plan_create": (C.c_int, [_P, _P, C.c_int, C.c_int, _P, _u64, _PP]),
    "cb_plan_create_parts": (C.c_int, [_P, _u32, C.c_int, C.c_int, _P, _u64, _PP]),
    "cb_plan_destroy": (None, [_P]),
    "cb_plan_num_parts": (C.c_int, [_P, C.POINTER(_u32)]),
    "cb_plan_stream": (C.c_void_p, [_P]),
    "cb_sample": (C.c_int, [_P, C.c_int, _P, _P, C.POINTER(Sched)]),
    "cb_sample_sync": (C.c_int, [_P, C.c_int, _P, _P, C.POINTER(Sched)]),
    "cb_sample_multi": (C.c_int, [_P, _P, _P, C.POINTER(Sched)]),
    "cb_plan_set_variate_table": (C.c_int, [_P, _P, C.c_int]),
    "cb_plan_set_layer_base": (C.c_int, [_P, C.c_int]),
    "cb_sample_device": (C.c_int, [_P, C.c_int, _P, _P, C.POINTER(Sched)]),
    "cb_gather": (C.c_int, [_P, _P]),
    "cb_synchronize": (C.c_int, [_P]),
    "cb_layer_sizes": (C.c_int, [_P, _u32, C.c_int, _P]),
    "cb_download_block": (C.c_int, [_P, _u32, C.c_int, _P, _P, _P, _P]),
    "cb_owner_set_size": (C.c_int, [_P, _u32, C.POINTER(_u64)]),
    "cb_plan_result_bytes": (C.c_int, [_P, _u32, _u64, C.POINTER(_u64)]),
    "cb_plan_result_async": (C.c_int, [_P, _u32, _P, _u64]),
    "cb_plan_result_copy": (C.c_int, [_P, _u32, _P, _u64, C.POINTER(_u64)]),
    "cb_plan_result_pack": (C.c_int, [_P, _u32]),
    "cb_download_owner_set": (C.c_int, [_P, _u32, _P]),
    "cb_download_exchange": (C.c_int, [_P, C.c_int, _P, _P, _P, _P]),
    "cb_download_rows": (C.c_int, [_P, _u32, _P]),
    "cb_rows_device": (C.c_int, [_P, _u32, _PP, C.POINTER(_u64)]),
    "cb_plan_capture": (C.c_int, [_P, C.c_int, _P, _P, C.POINTER(Sched)]),
    "cb_plan_replay": (C.c_int, [_P, _P, C.c_int, C.POINTER(Sched), C.c_int]),
    "cb_plan_create_dist": (C.c_int, [_P, _u32, C.c_int, C.c_int, _P, _u64, _PP]),
    "cb_plan_sample_layer": (C.c_int, [_P, C.c_int, _P, _u64, C.POINTER(Sched),
                                       C.POINTER(_u64)]),
    "cb_plan_layer_src": (C.c_int, [_P, C.c_int, _PP]),
    "cb_bucket_by_owner": (C.c_int, [_P, _P, _u64, _P, _u32, _P, _P, _P]),
    "cb_merge_owned": (C.c_int, [_P, C.c_int, _P, _u64, _P, _u64, C.POINTER(_u64), _P]),
    "cb_scatter_u32": (C.c_int, [_P, _P, _P, _u64, _P]),
    "cb_scatter_rows": (C.c_int, [_P, _P, _P, _u64, _u64, _P]),
    "cb_features_synth_shard": (C.c_int, [_P, _P, _u32, _u32, C.c_int, _u64, _PP]),
    "cb_gather_rows": (C.c_int, [_P, _P, _u64, _P, _P]),
    "cb_memcpy": (C.c_int, [_P, _P, _u64, C.c_int]),
    "cb_plan_profile": (C.c_int, [_P, C.c_int, _P, _P, C.POINTER(Sched), _P, _P, C.c_int,
                                  C.POINTER(C.c_int)]),
    "cb_plan_graph_profile": (C.c_int, [_P, _P, C.POINTER(Sched), _P, C.c_int,
                                        C.POINTER(C.c_int)]),
    "cb_plan_trace": (C.c_int, [_P, _P, _u64]),
    "cb_plan_launch_count": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(_u64)]),
    "cb_plan_captured_launches": (C.c_int, [_P, C.c_int, C.POINTER(_u64)]),
    "cb_cache_create": (C.c_int, [C.c_int, _u64, _u64, _u64, _PP]),
    "cb_cache_destroy": (None, [_P]),
    "cb_cache_access_trace": (C.c_int, [_P, _P, _u64, _P]),
    "cb_cache_access_ids": (C.c_int, [_P, _P, _u64, _u64, _P, _u32, _P, _P,
                                      C.POINTER(_u64), _P]),
    "cb_cache_access_plan": (C.c_int, [_P, _P, _u32, _u64, _P, _u32, _P, _P,
                                       C.POINTER(_u64)]),
    "cb_cache_access_host_ids": (C.c_int, [_P, _P, _u64, _u64, _P, _u32, C.POINTER(_u64)]),
    "cb_cache_stats": (C.c_int, [_P, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64)]),
    "cb_cache_reset_counters": (C.c_int, [_P]),
    "cb_cache_resident": (C.c_int, [_P, _P, _u64, C.POINTER(_u64)]),
    "cb_cache_storage": (C.c_int, [_P, _PP]),
    "cb_ccache_create": (C.c_int, [C.c_int, _u64, _u32, _u64, _PP]),
    "cb_ccache_destroy": (None, [_P]),
    "cb_ccache_gather_plan": (C.c_int, [_P, _P, _u32, _P]),
    "cb_ccache_stats": (C.c_int, [_P, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64)]),
    "cb_stack_fingerprint": (C.c_int, [_P, _u32, C.POINTER(_u64)]),
    "cb_shuffled_order": (C.c_int, [_u64, _u64, _P]),
    "cb_features_set_tier": (C.c_int, [_P, C.c_int]),
    "cb_kernel_launches": (C.c_int, [C.POINTER(_u64)]),
    "cb_gcn_model_init": (C.c_int, [C.c_int, _u32, _u32, _u32, C.c_int, _u64, _PP]),
    "cb_gcn_model_weights": (C.c_int, [_P, C.c_int, _P, C.c_int, C.POINTER(_u64),
                                       C.POINTER(_u64)]),
    "cb_gcn_model_destroy": (None, [_P]),
    "cb_train_step": (C.c_int, [_P, _P, _u32, _P, C.POINTER(C.c_double), _P]),
    "cb_plan_set_rw": (C.c_int, [_P, _u32, C.c_double, _u32]),
    "cb_plan_set_guard": (C.c_int, [_P, C.c_double, C.c_int, C.c_int]),
    "cb_plan_resolve_stats": (C.c_int, [_P, C.POINTER(_u64), C.POINTER(_u64)]),
    "cb_plan_meta_async": (C.c_int, [_P, _P, C.POINTER(_u64)]),
    "cb_px_setup": (C.c_int, [_P, _P, _u32, _P]),
    "cb_px_connect": (C.c_int, [_P, _u32, _P]),
    "cb_px_layer": (C.c_int, [_P, C.c_int, _P, _u64, C.POINTER(Sched)]),
    "cb_px_owner": (C.c_int, [_P, C.c_int]),
    "cb_px_locate": (C.c_int, [_P, C.c_int]),
    "cb_px_finish": (C.c_int, [_P]),
    "cb_px_barrier": (C.c_int, [_P]),
    "cb_px_setup_staging": (C.c_int, [_P, _P, _P]),
    "cb_px_connect_staging": (C.c_int, [_P, _u32, _P]),
    "cb_px_set_cache": (C.c_int, [_P, _P]),
    "cb_px_set_requester_cache": (C.c_int, [_P, _P]),
    "cb_px_set_clock_cache": (C.c_int, [_P, _P]),
    "cb_px_requester_stats": (C.c_int, [_P, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64)]),
    "cb_px_gather_cached": (C.c_int, [_P, _u64, C.POINTER(_u64), C.POINTER(_u64),
                                      C.POINTER(_u64)]),
    "cb_px_capture": (C.c_int, [_P, _u64, C.POINTER(Sched), _P]),
    "cb_px_replay": (C.c_int, [_P, _P, C.c_int, C.POINTER(Sched)]),
    "cb_px_sizes": (C.c_int, [_P, C.c_int, C.POINTER(_u64), C.POINTER(_u64)]),
    "cb_px_download": (C.c_int, [_P, C.c_int, _P, _P, _P, _P]),
    "cb_features_export": (C.c_int, [_P, _P, C.POINTER(_u64)]),
    "cb_px_connect_features": (C.c_int, [_P, _u32, _P, _u64, _P]),
    "cb_px_gather": (C.c_int, [_P, _P]),
    "cb_plan_input_ids": (C.c_int, [_P, _u32, _PP, C.POINTER(_u64)]),
}

_lib = None


def header_symbols() -> list[str]:
    """Every cb_* entry point declared in include/coopbatch_cuda.h."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(cb_[a-z0-9_]+)\s*\(", txt)))


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the CUDA extension is not built "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`). "
            "There is no CPU fallback.")
    L = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L
