"""ctypes binding of libgts.so (the C ABI declared in include/gts.h).

The product path has no CPU fallback: if the shared library is missing or
no CUDA device is visible, calls raise instead of computing elsewhere.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgts.so")

GTS_OK, GTS_EINVAL, GTS_EBUDGET, GTS_EMETRIC, GTS_ECUDA, GTS_EOOM, GTS_EREBUILD = range(7)
FLAG_PRUNING, FLAG_CACHE = 1, 2

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)


class GtsDataset(C.Structure):
    _fields_ = [
        ("metric", C.c_int32), ("n", C.c_int64), ("dim", C.c_int64),
        ("vectors", _f64p), ("codes", _i32p), ("offsets", _i64p), ("ids", _i64p),
    ]


class GtsTree(C.Structure):
    _fields_ = [
        ("nc", C.c_int64), ("levels", C.c_int64), ("split_rounds", C.c_int64),
        ("nodes", C.c_int64), ("n", C.c_int64),
        ("pivot_id", _i64p), ("pivot_row", _i64p), ("pos", _i64p), ("size", _i64p),
        ("min_dis", _f64p), ("max_dis", _f64p),
        ("rows", _i64p), ("dis", _f64p), ("tombstone", _u8p),
    ]


class GtsQueryBatch(C.Structure):
    _fields_ = [
        ("metric", C.c_int32), ("nq", C.c_int64), ("dim", C.c_int64),
        ("vectors", _f64p), ("codes", _i32p), ("offsets", _i64p),
    ]


_lib = None
_lock = threading.Lock()


def lib():
    """Load libgts.so (building it first if the sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            from . import _build
            _build.build()
        L = C.CDLL(LIB_PATH)
        v = C.c_void_p
        sig = {
            "gts_tree_height": (C.c_int, [C.c_int64, C.c_int64, _i64p, _i64p]),
            "gts_node_count": (C.c_int64, [C.c_int64, C.c_int64]),
            "gts_build_tree": (C.c_int, [C.POINTER(GtsDataset), C.c_int64, C.c_int, C.POINTER(GtsTree)]),
            "gts_index_create": (C.c_int, [C.POINTER(GtsDataset), C.POINTER(GtsTree), C.c_int, C.POINTER(v)]),
            "gts_index_destroy": (C.c_int, [v]),
            "gts_index_set_tombstones": (C.c_int, [v, _u8p, v]),
            "gts_queries_upload": (C.c_int, [v, C.POINTER(GtsQueryBatch), v, C.POINTER(v)]),
            "gts_queries_free": (C.c_int, [v]),
            "gts_range_batch": (C.c_int, [v, v, _f64p, C.c_int64, C.c_int, v, C.POINTER(v)]),
            "gts_knn_batch": (C.c_int, [v, v, _i64p, C.c_int64, C.c_int, v, C.POINTER(v)]),
            "gts_range_batch_host": (C.c_int, [v, C.POINTER(GtsQueryBatch), _f64p, C.c_int64, C.c_int, v, C.POINTER(v)]),
            "gts_knn_batch_host": (C.c_int, [v, C.POINTER(GtsQueryBatch), _i64p, C.c_int64, C.c_int, v, C.POINTER(v)]),
            "gts_batch_host": (C.c_int, [v, C.POINTER(GtsQueryBatch), C.c_int, _f64p, _i64p, C.c_int64, C.c_int,
                                         v, C.POINTER(v)]),
            "gts_index_cache_set": (C.c_int, [v, C.POINTER(GtsDataset), v]),
            "gts_result_info": (C.c_int, [v, _i64p, _i64p, _i64p, _i64p]),
            "gts_result_copy": (C.c_int, [v, _i64p, _i64p, _f64p, _i64p, _i64p, v]),
            "gts_result_device": (C.c_int, [v, C.POINTER(v), C.POINTER(v), C.POINTER(v)]),
            "gts_result_free": (C.c_int, [v]),
            "gts_pair_distances": (C.c_int, [C.c_int32, C.c_int64, C.c_int64, _f64p, _f64p, _i32p, _i64p,
                                             _i32p, _i64p, _f64p, v]),
            "gts_knn_probe": (C.c_int, [v, v, _i64p, v, v]),
            "gts_knn_batch_bounded": (C.c_int, [v, v, _i64p, v, C.c_int64, C.c_int, v, C.POINTER(v)]),
            "gts_merge_results": (C.c_int, [C.c_int, C.c_int64, v, v, v, v, v, v, v, C.POINTER(v)]),
            "gts_multi_create": (C.c_int, [C.c_int, C.POINTER(v), C.POINTER(v)]),
            "gts_multi_destroy": (C.c_int, [v]),
            "gts_multi_batch_host": (C.c_int, [v, C.POINTER(GtsQueryBatch), C.c_int, _f64p, _i64p, C.c_int64,
                                               C.c_int, C.POINTER(v)]),
            "gts_build_tree_device": (C.c_int, [C.POINTER(GtsDataset), C.c_int64, C.c_int, C.POINTER(GtsTree)]),
            "gts_build_tree_device_f32": (C.c_int, [C.c_int32, C.c_int64, C.c_int64, v, _i64p, C.c_int64, C.c_int,
                                                    C.POINTER(GtsTree)]),
            "gts_index_create_f32dev": (C.c_int, [C.POINTER(GtsTree), C.c_int32, C.c_int64, v, _i64p, C.c_int,
                                                  C.POINTER(v)]),
            "gts_generate_clustered": (C.c_int, [C.c_uint64, C.c_int64, C.c_int64, C.c_int64, C.c_float, C.c_int64,
                                                 C.c_int64, C.c_uint64, C.c_float, v, v]),
            "gts_index_insert": (C.c_int, [v, C.POINTER(GtsDataset), _i32p, v]),
            "gts_index_erase": (C.c_int, [v, _i32p, C.c_int64, v]),
            "gts_launch_count": (C.c_int64, []),
            "gts_device_count": (C.c_int, []),
            "gts_profile_enable": (C.c_int, [C.c_int]),
            "gts_profile_read": (C.c_int, [C.c_char_p, C.c_int64, C.c_int]),
            "gts_bench_int_peak": (C.c_int, [_f64p, v]),
            "gts_bench_fp32_peak": (C.c_int, [_f64p, v]),
            "gts_last_error": (C.c_char_p, []),
            "gts_version": (C.c_char_p, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        return _lib


EXPORTED = (
    "gts_tree_height", "gts_node_count", "gts_build_tree", "gts_index_create", "gts_index_destroy",
    "gts_index_set_tombstones", "gts_queries_upload", "gts_queries_free", "gts_range_batch",
    "gts_knn_batch", "gts_range_batch_host", "gts_knn_batch_host", "gts_result_info", "gts_result_copy",
    "gts_result_device", "gts_result_free", "gts_pair_distances", "gts_launch_count", "gts_last_error",
    "gts_version", "gts_profile_enable", "gts_profile_read", "gts_bench_int_peak", "gts_batch_host",
    "gts_index_cache_set", "gts_knn_probe", "gts_knn_batch_bounded", "gts_merge_results", "gts_multi_create",
    "gts_multi_destroy", "gts_multi_batch_host", "gts_build_tree_device", "gts_build_tree_device_f32",
    "gts_index_create_f32dev", "gts_generate_clustered", "gts_bench_fp32_peak",
    "gts_device_count", "gts_index_insert", "gts_index_erase",
)


def profile_read(reset=True):
    import json
    buf = C.create_string_buffer(1 << 16)
    check(lib().gts_profile_read(buf, len(buf), int(reset)))
    return json.loads(buf.value.decode())


def check(rc: int) -> None:
    """Raise the reference's exception type for a non-zero status."""
    if rc == GTS_OK:
        return
    msg = lib().gts_last_error().decode(errors="replace")
    from .metrics import MetricMismatchError
    from .runtime import BudgetError
    if rc == GTS_EINVAL:
        raise ValueError(msg)
    if rc == GTS_EBUDGET:
        raise BudgetError(msg)
    if rc == GTS_EMETRIC:
        raise MetricMismatchError(msg)
    if rc == GTS_EOOM:
        raise MemoryError(msg)
    raise RuntimeError(f"libgts: {msg}")


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def launch_count() -> int:
    return int(lib().gts_launch_count())
