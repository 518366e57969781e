"""ctypes binding of the in-tree native library (include/tokenselect.h).

The library is the product: there is no Python or CPU implementation behind
these calls. If the .so is missing this module raises at import time.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# TS_LIB_PATH: an alternative build of the same library (dev A/B timing)
LIB_PATH = os.environ.get("TS_LIB_PATH") or os.path.join(HERE, "_build", "libtokenselect.so")

_sz = C.c_size_t
_p = C.c_void_p
_u32p = C.POINTER(C.c_uint32)


class TsStatus:
    OK, INVALID_ARGUMENT, OUT_OF_RANGE, CAPACITY, CUDA_ERROR = range(5)


class EngineConfig(C.Structure):
    """ts_engine_config == EngineConfig (attention.hpp:12-27)."""

    _fields_ = [
        ("k", _sz),
        ("n_local", _sz),
        ("n_init", _sz),
        ("chunk_size", _sz),
        ("theta", C.c_double),
        ("num_heads", _sz),
        ("num_kv_heads", _sz),
        ("head_dim", _sz),
        ("block_size", _sz),
        ("selection_method", C.c_int),
    ]


# name -> (restype, argtypes)
SIGNATURES = {
    "ts_last_error": (C.c_char_p, []),
    "ts_version": (C.c_char_p, []),
    "ts_launch_count": (C.c_uint64, []),
    "ts_engine_config_default": (None, [C.POINTER(EngineConfig)]),
    "ts_engine_config_validate": (C.c_int, [C.POINTER(EngineConfig)]),
    "ts_pool_create": (C.c_int, [_sz, _sz, _sz, _sz, C.POINTER(_p)]),
    "ts_pool_destroy": (None, [_p]),
    "ts_pool_create_sequence": (C.c_int, [_p, C.POINTER(C.c_uint32)]),
    "ts_pool_append_kv": (C.c_int, [_p, C.c_uint32, _p, _p, _sz, C.POINTER(_sz), C.POINTER(_sz)]),
    "ts_pool_append_kv_bf16": (C.c_int, [_p, C.c_uint32, _p, _p, _sz, C.POINTER(_sz), C.POINTER(_sz)]),
    "ts_pool_gather": (C.c_int, [_p, C.c_uint32, _p, _sz, _p, _p]),
    "ts_pool_release": (C.c_int, [_p, C.c_uint32]),
    "ts_pool_logical_len": (C.c_int, [_p, C.c_uint32, C.POINTER(_sz)]),
    "ts_pool_shuffle_free_frames": (C.c_int, [_p, C.c_uint64]),
    "ts_pool_page_table_json": (C.c_int, [_p, C.c_uint32, C.c_char_p, _sz, C.POINTER(_sz)]),
    "ts_pool_total_frames": (_sz, [_p]),
    "ts_pool_free_frames": (_sz, [_p]),
    "ts_pool_page_size": (_sz, [_p]),
    "ts_pool_num_kv_heads": (_sz, [_p]),
    "ts_pool_head_dim": (_sz, [_p]),
    "ts_pool_device_views": (C.c_int, [_p, C.c_uint32, C.POINTER(_p), C.POINTER(_p), C.POINTER(_p)]),
    "ts_score_paged": (C.c_int, [_p, C.c_uint32, _p, _sz, _sz, _p, _sz, _sz, _p]),
    "ts_select": (C.c_int, [_p, _sz, _sz, _p, _sz, C.c_int, _p, _p, C.POINTER(_sz)]),
    "ts_select_for_chunk": (C.c_int, [_p, C.c_uint32, _p, _sz, _sz, _p, _sz, _sz, C.c_int, _sz, _p, _p,
                                      C.POINTER(_sz)]),
    "ts_sparse_attend": (C.c_int, [_p, C.c_uint32, _p, _p, _p, _sz, _sz, _p, _sz, _p, _sz, _p, _sz, _p]),
    "ts_engine_create": (C.c_int, [C.POINTER(EngineConfig), _sz, _sz, C.POINTER(_p)]),
    "ts_engine_create_layers": (C.c_int, [C.POINTER(EngineConfig), _sz, _sz, _sz, C.POINTER(_p)]),
    "ts_engine_set_layer": (C.c_int, [_p, _sz]),
    "ts_engine_num_layers": (_sz, [_p]),
    "ts_engine_destroy": (None, [_p]),
    "ts_engine_set_stream": (C.c_int, [_p, _p]),
    "ts_engine_append": (C.c_int, [_p, _sz, _p, _p, _sz]),
    "ts_engine_append_bf16": (C.c_int, [_p, _sz, _p, _p, _sz]),
    "ts_engine_prefill": (C.c_int, [_p, _sz, _p, _p, _p, _sz, _p, _p, _p, _sz]),
    "ts_engine_prefill_async": (C.c_int, [_p, _sz, _p, _p, _p, _sz, _p]),
    "ts_engine_decode": (C.c_int, [_p, _p, _p, _p, _p, _p, _p, _p]),
    "ts_engine_decode_async": (C.c_int, [_p, _p, _p, _p, _p]),
    "ts_engine_force_miss": (C.c_int, [_p, _sz]),
    "ts_engine_set_theta": (C.c_int, [_p, _sz, C.c_double]),
    "ts_engine_set_trace": (C.c_int, [_p, C.c_int]),
    "ts_engine_read_trace": (C.c_int, [_p, _p, _sz]),
    "ts_engine_stats": (C.c_int, [_p, _sz, C.POINTER(_sz), C.POINTER(_sz), C.POINTER(_sz), C.POINTER(C.c_int),
                                  C.POINTER(C.c_double)]),
    "ts_engine_cached_selection": (C.c_int, [_p, _sz, _p, _p, C.POINTER(_sz)]),
    "ts_engine_sync": (C.c_int, [_p]),
    "ts_engine_cache_entry": (C.c_int, [_p, _sz, _p, C.POINTER(C.c_int), C.POINTER(C.c_double)]),
    "ts_shard_engine_create": (C.c_int, [C.POINTER(EngineConfig), _sz, C.c_int, C.c_int, C.POINTER(_p)]),
    "ts_shard_stats": (C.c_int, [_p, _p, _p, _p, _sz, _sz, _p]),
    "ts_shard_select": (C.c_int, [_p, _p, _p]),
    "ts_shard_attend": (C.c_int, [_p, _p, _p, _p]),
    "ts_shard_combine": (C.c_int, [_p, _p, C.c_int, _sz, _sz, _p, _p]),
    "ts_shard_combine_packed": (C.c_int, [_p, C.c_int, _sz, _sz, _p, _p]),
    "ts_softmax_rows": (C.c_int, [_p, _sz, _sz, _p]),
    "ts_topk_indices": (C.c_int, [_p, _sz, _sz, _p, C.POINTER(_sz)]),
    "ts_cosine": (C.c_int, [_p, _p, _sz, C.POINTER(C.c_double)]),
    "ts_chunk_mean": (C.c_int, [_p, _sz, _sz, _p]),
    "ts_sdpa_full": (C.c_int, [_p, _sz, _sz, _p, _p, _sz, _sz, _sz, _p]),
    "ts_comm_unique_id": (C.c_int, [_p]),
    "ts_comm_create": (C.c_int, [_p, C.c_int, C.c_int, C.POINTER(_p)]),
    "ts_comm_destroy": (None, [_p]),
    "ts_shard_decode_step": (C.c_int, [_p, _p, _p, _p, _p, _sz, _sz, _p]),
    "ts_engine_pool": (_p, [_p]),
    "ts_engine_sequence": (C.c_uint32, [_p, _sz]),
}


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"native library {path} is missing: run `python -m paper_2411_02886_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = load()


class CapacityError(RuntimeError):
    """selattn::capacity_error (kv_pool.hpp:15-17)."""


def check(rc: int) -> None:
    if rc == TsStatus.OK:
        return
    msg = lib.ts_last_error().decode()
    if rc == TsStatus.INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument -> ValueError (pybind11 mapping)
    if rc == TsStatus.OUT_OF_RANGE:
        raise IndexError(msg)  # std::out_of_range -> IndexError
    if rc == TsStatus.CAPACITY:
        raise CapacityError(msg)
    raise RuntimeError(msg)
