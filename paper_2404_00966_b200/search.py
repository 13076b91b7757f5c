"""Batch exact range / kNN search on the GPU -- drop-in for the reference's
`metrictree.search` (search.py:28-570).

`BatchSearcher(tree, runtime=None, memory_units=None, pruning=True)` keeps
the reference's constructor, `range_batch` / `knn_batch` signatures, return
values ((ids, distances) per query, sorted by (distance, id), plus
SearchStats) and error types.  Underneath, one C-ABI call runs the whole
batch on the device (csrc/engine.cu).  Array surfaces `range_batch_array` /
`knn_batch_array` return CSR results without per-query Python objects.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .metrics import METRIC_CODES, STRING_METRICS
from .runtime import DEFAULT_MEMORY_UNITS, BudgetError

# memory_units=HBM_SIZED: the device default, sized to free HBM (csrc/engine.cu
# hbm_rows); None keeps the reference's DEFAULT_MEMORY_UNITS (runtime.py:18),
# so a default-constructed searcher logs the reference's size_limits
HBM_SIZED = -1
DEVICE_MEMORY_UNITS = HBM_SIZED

RANGE = "range"
KNN = "knn"


# -- predicates and scheduling helpers (reference search.py:28-95) ---------

def object_prunable(entry_dis, dqp, radius):
    return abs(entry_dis - dqp) > radius


def node_prunable_range(dqp, radius, min_dis, max_dis):
    return dqp + radius < min_dis or dqp - radius > max_dis


def node_prunable_knn(dqp, bound, min_dis, max_dis):
    return dqp + bound <= min_dis or dqp - bound >= max_dis


def current_kth_bound(sorted_dis, k):
    if k < 1:
        raise ValueError("k must be >= 1")
    arr = np.asarray(sorted_dis, dtype=np.float64)
    return float(arr[k - 1]) if arr.size >= k else float("inf")


def level_size_limit(capacity, node_capacity, split_rounds, layer):
    """max(1, capacity // ((split_rounds - layer + 1) * node_capacity))."""
    if not 1 <= layer <= split_rounds:
        raise ValueError(f"layer {layer} outside [1, {split_rounds}]")
    return max(1, capacity // ((split_rounds - layer + 1) * node_capacity))


def compute_query_groups(row_counts, size_limit):
    """Greedy first-fit grouping (search.py:73-95)."""
    groups, loads = [], []
    for q, count in enumerate(row_counts):
        for g, load in enumerate(loads):
            if load + count <= size_limit:
                groups[g].append(q)
                loads[g] = load + count
                break
        else:
            groups.append([q])
            loads.append(count)
    return groups


class SearchStats:
    """Per-query work counters for one batch call (search.py:98-113)."""

    def __init__(self, nq):
        self.verified = np.zeros(nq, dtype=np.int64)
        self.pruned_nodes = np.zeros(nq, dtype=np.int64)
        self.size_limits = {}
        self.peak_units = 0

    @property
    def total_verified(self):
        return int(self.verified.sum())

    @property
    def total_pruned(self):
        return int(self.pruned_nodes.sum())


class CsrResult:
    """Host CSR answers: query q owns ids/dis[offsets[q]:offsets[q+1]]."""

    def __init__(self, offsets, ids, dis, stats):
        self.offsets, self.ids, self.dis, self.stats = offsets, ids, dis, stats

    def answers(self):
        o = self.offsets
        return [(self.ids[o[q]:o[q + 1]], self.dis[o[q]:o[q + 1]]) for q in range(o.size - 1)]


def _fetch(res_handle, nq):
    L = _lib.lib()
    try:
        n = C.c_int64()
        tot = C.c_int64()
        peak = C.c_int64()
        limits = np.zeros(64, dtype=np.int64)
        _lib.check(L.gts_result_info(res_handle, C.byref(n), C.byref(tot), C.byref(peak),
                                     _lib.ptr(limits, _lib._i64p)))
        offsets = np.zeros(nq + 1, dtype=np.int64)
        ids = np.empty(max(tot.value, 1), dtype=np.int64)
        dis = np.empty(max(tot.value, 1), dtype=np.float64)
        stats = SearchStats(nq)
        _lib.check(L.gts_result_copy(res_handle, _lib.ptr(offsets, _lib._i64p), _lib.ptr(ids, _lib._i64p),
                                     _lib.ptr(dis, _lib._f64p), _lib.ptr(stats.verified, _lib._i64p),
                                     _lib.ptr(stats.pruned_nodes, _lib._i64p), None))
        stats.peak_units = int(peak.value)
        stats.size_limits = {int(l): int(limits[l]) for l in range(64) if limits[l]}
        return CsrResult(offsets, ids[:tot.value], dis[:tot.value], stats)
    finally:
        L.gts_result_free(res_handle)


class BatchSearcher:
    """Exact batch query engine over one FlatPivotTree, on the GPU.

    Args mirror the reference (search.py:214-234): tree, runtime (accepted,
    unused: the device does the parallel work), memory_units (row budget of
    the one materialized frontier table; None = the reference's default of
    1<<20 rows, HBM_SIZED = the device default sized to free HBM), pruning.
    """

    def __init__(self, tree, runtime=None, memory_units=None, pruning=True, device=0, _use_cache=False):
        self._use_cache = _use_cache
        self.tree = tree
        self.ds = tree.dataset
        self.rt = runtime
        self.capacity = DEFAULT_MEMORY_UNITS if memory_units is None else int(memory_units)
        self.pruning = pruning
        self.device = device
        if tree.n > 0 and self.capacity != HBM_SIZED and self.capacity < tree.nc:
            raise BudgetError(f"memory_units {self.capacity} below fan-out {tree.nc}")

    # -- public API (search.py:238-260) -------------------------------------

    def range_batch(self, payloads, radii):
        res = self.range_batch_array(payloads, radii)
        return res.answers(), res.stats

    def knn_batch(self, payloads, ks):
        res = self.knn_batch_array(payloads, ks)
        return res.answers(), res.stats

    @staticmethod
    def _broadcast(value, nq, what):
        arr = np.atleast_1d(np.asarray(value, dtype=np.float64))
        if arr.size == 1:
            return np.full(nq, float(arr[0]))
        if arr.size != nq:
            raise ValueError(f"{what} list length {arr.size} != {nq} queries")
        return arr.astype(np.float64)

    # -- array surfaces -----------------------------------------------------

    def range_batch_array(self, payloads, radii):
        nq = len(payloads)
        radii = np.ascontiguousarray(self._broadcast(radii, nq, "radius"))
        if np.any(radii < 0):
            raise ValueError("radius must be >= 0")
        return self._run(RANGE, payloads, radii, None)

    def knn_batch_array(self, payloads, ks):
        nq = len(payloads)
        ks = np.ascontiguousarray(self._broadcast(ks, nq, "k").astype(np.int64))
        if np.any(ks < 1):
            raise ValueError("k must be >= 1")
        return self._run(KNN, payloads, None, ks)

    def _batch_struct(self, payloads):
        """Validated C query batch + arrays to keep alive."""
        prepared = self.ds.prepare_batch(payloads)
        code = METRIC_CODES[self.ds.metric]
        if self.ds.metric in STRING_METRICS:
            codes, off = prepared
            codes = codes if codes.size else np.zeros(1, np.int32)
            qb = _lib.GtsQueryBatch(code, len(payloads), 0, None, _lib.ptr(codes, _lib._i32p),
                                    _lib.ptr(off, _lib._i64p))
            return qb, (codes, off)
        mat = np.ascontiguousarray(prepared, dtype=np.float64)
        if mat.size == 0:
            mat = np.zeros((len(payloads), self.ds.dim or 1))
        qb = _lib.GtsQueryBatch(code, len(payloads), self.ds.dim or mat.shape[1], _lib.ptr(mat, _lib._f64p),
                                None, None)
        return qb, (mat,)

    def _run(self, mode, payloads, radii, ks):
        tree = self.tree
        nq = len(payloads)
        if nq == 0 or tree.levels == 0:
            # validate payloads even when there is nothing to search
            if nq:
                self.ds.prepare_batch(payloads)
            stats = SearchStats(nq)
            return CsrResult(np.zeros(nq + 1, dtype=np.int64), np.empty(0, np.int64), np.empty(0), stats)
        qb, keep = self._batch_struct(payloads)
        dev = tree.device_index(self.device)
        L = _lib.lib()
        h = C.c_void_p()
        flags = (_lib.FLAG_PRUNING if self.pruning else 0) | (_lib.FLAG_CACHE if self._use_cache else 0)
        rc = L.gts_batch_host(dev.h, C.byref(qb), 0 if mode == RANGE else 1,
                              _lib.ptr(radii, _lib._f64p) if radii is not None else None,
                              _lib.ptr(ks, _lib._i64p) if ks is not None else None,
                              max(self.capacity, 0), flags, None, C.byref(h))
        _lib.check(rc)
        return _fetch(h, nq)
