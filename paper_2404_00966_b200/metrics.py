"""Metric kinds and exact pair distances (reference metrics.py:15-223).

Pair distances run on the device (`gts_pair_distances`): float64 in numpy's
row-sum order for L1/L2, the exact integer for edit distance.
"""

from __future__ import annotations

import numpy as np

EDIT = "edit"
L1 = "l1"
L2 = "l2"
ANGULAR = "angular"

METRIC_KINDS = (EDIT, L1, L2, ANGULAR)
VECTOR_METRICS = (L1, L2, ANGULAR)
STRING_METRICS = (EDIT,)

# C-ABI metric codes (include/gts.h; = reference io.py:30-35)
METRIC_CODES = {EDIT: 0, L1: 1, L2: 2, ANGULAR: 3}


class MetricMismatchError(TypeError):
    """Payload is incompatible with the requested metric (metrics.py:25-26)."""


def _require_kind(metric):
    if metric not in METRIC_KINDS:
        raise MetricMismatchError(f"unknown metric kind: {metric!r}")


def encode_string(s):
    """UTF-32 code points of a str (metrics.py:34-38)."""
    if not isinstance(s, str):
        raise MetricMismatchError(f"expected str payload, got {type(s).__name__}")
    return np.frombuffer(s.encode("utf-32-le"), dtype=np.int32)


def as_vector(v):
    """1-D float64 array of finite values (metrics.py:41-51)."""
    try:
        arr = np.asarray(v, dtype=np.float64)
    except (TypeError, ValueError) as exc:
        raise MetricMismatchError(f"payload is not numeric: {exc}") from exc
    if arr.ndim != 1:
        raise MetricMismatchError(f"expected 1-D vector payload, got ndim={arr.ndim}")
    if not np.all(np.isfinite(arr)):
        raise MetricMismatchError("vector payload contains non-finite values")
    return arr


def pack_strings(strings):
    """(codes int32, offsets int64[n+1]) of a list of str."""
    lens = np.fromiter((len(s) for s in strings), dtype=np.int64, count=len(strings))
    off = np.zeros(len(strings) + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    if len(strings):
        codes = np.frombuffer("".join(strings).encode("utf-32-le"), dtype=np.int32)
    else:
        codes = np.empty(0, dtype=np.int32)
    return np.ascontiguousarray(codes), off


def pair_distances(metric, a, b):
    """Distances of aligned payload pairs a[i], b[i] on the device."""
    from . import _lib
    import ctypes as C
    _require_kind(metric)
    L = _lib.lib()
    n = len(a)
    out = np.empty(n, dtype=np.float64)
    if n == 0:
        return out
    if metric == EDIT:
        ca, oa = pack_strings(list(a))
        cb, ob = pack_strings(list(b))
        ca = ca if ca.size else np.zeros(1, np.int32)
        cb = cb if cb.size else np.zeros(1, np.int32)
        _lib.check(L.gts_pair_distances(0, n, 0, None, None, _lib.ptr(ca, _lib._i32p), _lib.ptr(oa, _lib._i64p),
                                        _lib.ptr(cb, _lib._i32p), _lib.ptr(ob, _lib._i64p),
                                        _lib.ptr(out, _lib._f64p), None))
        return out
    A = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    B = np.ascontiguousarray(np.asarray(b, dtype=np.float64))
    if A.shape != B.shape or A.ndim != 2:
        raise MetricMismatchError("vector dimensionality mismatch")
    _lib.check(L.gts_pair_distances(METRIC_CODES[metric], n, A.shape[1], _lib.ptr(A, _lib._f64p),
                                    _lib.ptr(B, _lib._f64p), None, None, None, None,
                                    _lib.ptr(out, _lib._f64p), C.c_void_p(0)))
    return out


def edit_distance(a, b):
    """Unit-cost edit distance (metrics.py:102-104)."""
    encode_string(a)
    encode_string(b)
    return float(pair_distances(EDIT, [a], [b])[0])


def distance(metric, a, b):
    """Distance between two raw payloads (metrics.py:196-223)."""
    _require_kind(metric)
    if metric == EDIT:
        return edit_distance(a, b)
    va = as_vector(a)
    vb = as_vector(b)
    if va.shape != vb.shape:
        raise MetricMismatchError(f"vector dimensionality mismatch: {va.shape[0]} vs {vb.shape[0]}")
    return float(pair_distances(metric, va[None, :], vb[None, :])[0])
