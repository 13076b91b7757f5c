"""Multi-GPU sharding: one GTS tree per shard, the query batch replicated, the
per-shard answers exchanged and merged (BASELINE.json north_star; SURVEY.md
§8(e)).

Exact search over a partition is the union of exact per-shard answers
(Def. 1/2).  The reference has one index, so its anchors
are the merges it performs inside that index: `_KnnPool.merge` keeps the k
smallest (distance, id) (search.py:116-144) and `_collect` orders range
answers by (distance, id) (search.py:298-314).  Two surfaces:

* `ShardedIndex` -- one Python object over several shard indexes in one
  process (SURVEY.md §8(b) "device_mask": the list of devices).  One C-ABI
  call per batch (`gts_multi_batch_host`): a host thread per shard uploads
  the batch and searches on its device; kNN first exchanges every shard's
  probe radius (device MIN: each shard's radius bounds its own k-th
  distance, so the MIN bounds the global one and every shard prunes with
  it); the answers are gathered over NVLink peer copies and merged on the
  first shard's device by `k_merge_rank` (csrc/sharded.cuh).

* `ShardExchange` -- one process per GPU under torch.distributed (NCCL).
  Rank r owns the queries [bounds[r], bounds[r+1]).  kNN: `knn_bound`
  all-reduces the probe radii with MIN (nq x 4 B).  Answers: every rank
  sends each owner the CSR answers of the owner's queries
  (`all_to_all_single`, answers packed as 16-byte (id, distance bits)
  records), and the owner merges the world-size sorted lists of each of its
  queries on its device with `gts_merge_results` (k_merge_rank).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .search import CsrResult, SearchStats, BatchSearcher, DEVICE_MEMORY_UNITS, KNN, RANGE
from .runtime import BudgetError
from .tree import TreeConfig, build as build_tree


# ---------------------------------------------------------------------------
# device merge (libgts k_merge_rank) on torch tensors
# ---------------------------------------------------------------------------

def _vp(t):
    return C.c_void_p(t.data_ptr()) if t is not None and t.numel() else None


def device_merge(counts, ids, dis, ks=None, stream=None):
    """Merge S sorted per-source answer lists per query on the device.

    counts: int64 [S, nq] (device); ids int64 / dis float64: every source's
    answers, source-major then query-major.  ks: int64 [nq] (kNN: keep the k
    smallest) or None (range: keep all).  Returns (offsets, ids, dis) torch
    tensors on the same device, sorted by (distance, id) per query."""
    S, nq = counts.shape
    dev = counts.device
    L = _lib.lib()
    h = C.c_void_p()
    st = C.c_void_p(stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream)
    counts = counts.contiguous()
    ids = ids.contiguous()
    dis = dis.contiguous()
    _lib.check(L.gts_merge_results(int(S), int(nq), _vp(counts), _vp(ids), _vp(dis),
                                   _vp(ks) if ks is not None else None, None, None, st, C.byref(h)))
    try:
        tot = C.c_int64()
        _lib.check(L.gts_result_info(h, None, C.byref(tot), None, None))
        off = torch.empty(nq + 1, dtype=torch.int64, device=dev)
        oid = torch.empty(max(tot.value, 1), dtype=torch.int64, device=dev)
        odi = torch.empty(max(tot.value, 1), dtype=torch.float64, device=dev)
        _lib.check(L.gts_result_copy(h, C.cast(off.data_ptr(), _lib._i64p), C.cast(oid.data_ptr(), _lib._i64p),
                                     C.cast(odi.data_ptr(), _lib._f64p), None, None, st))
        return off, oid[:tot.value], odi[:tot.value]
    finally:
        L.gts_result_free(h)


# ---------------------------------------------------------------------------
# one process per GPU: owner-partitioned exchange over torch.distributed
# ---------------------------------------------------------------------------

class ShardExchange:
    """Exchange + merge of per-shard answers for one replicated query batch.

    `merge` defaults to the device merge; tests on CPU inject a host merge
    with the same contract to check the partitioning and the collectives."""

    def __init__(self, nq, device, group=None, merge=None):
        self.nq = int(nq)
        self.device = device
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.bounds = [self.nq * r // self.world for r in range(self.world + 1)]
        self.merge = merge or device_merge
        # gloo has no device collectives: stage through host memory there
        self.stage = dist.is_initialized() and dist.get_backend(group) == "gloo" and device.type == "cuda"

    @property
    def own(self):
        """This rank's query slice [lo, hi)."""
        return self.bounds[self.rank], self.bounds[self.rank + 1]

    def _a2a(self, out, inp, out_splits, in_splits):
        if self.world == 1:
            out.copy_(inp)
            return out
        if self.stage:
            o = out.cpu()
            dist.all_to_all_single(o, inp.cpu(), out_splits, in_splits, group=self.group)
            out.copy_(o)
            return out
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)
        return out

    def knn_bound(self, radius):
        """In place: radius[q] = MIN over shards (float32 [nq])."""
        if self.world > 1:
            if self.stage:
                r = radius.cpu()
                dist.all_reduce(r, op=dist.ReduceOp.MIN, group=self.group)
                radius.copy_(r)
            else:
                dist.all_reduce(radius, op=dist.ReduceOp.MIN, group=self.group)
        return radius

    def exchange(self, offsets, ids, dis):
        """Send every owner its queries' answers.  Returns (counts [W, nq_own],
        ids, dis) as received, source-major."""
        W, b = self.world, self.bounds
        lo, hi = self.own
        nown = hi - lo
        counts = offsets[1:] - offsets[:-1]
        rc = torch.empty(W * nown, dtype=torch.int64, device=offsets.device)
        self._a2a(rc, counts, [nown] * W, [b[o + 1] - b[o] for o in range(W)])
        cut = offsets[torch.tensor(b, device=offsets.device)].tolist()
        send = [cut[o + 1] - cut[o] for o in range(W)]
        rc = rc.view(W, nown)
        recv = rc.sum(dim=1).tolist()
        # one 16-byte record per answer: (id, distance bits)
        pack = torch.stack([ids[cut[0]:cut[-1]], dis[cut[0]:cut[-1]].view(torch.int64)], dim=1)
        out = torch.empty((sum(recv), 2), dtype=torch.int64, device=offsets.device)
        self._a2a(out, pack, recv, send)
        return rc, out[:, 0].contiguous(), out[:, 1].contiguous().view(torch.float64)

    def merge_range(self, offsets, ids, dis):
        rc, rid, rdi = self.exchange(offsets, ids, dis)
        return self.merge(rc, rid, rdi, None)

    def merge_knn(self, offsets, ids, dis, ks):
        """ks: int64 [nq] (the full batch's k values, on the device)."""
        rc, rid, rdi = self.exchange(offsets, ids, dis)
        lo, hi = self.own
        return self.merge(rc, rid, rdi, ks[lo:hi].contiguous())


def result_tensors(h, device, stream):
    """Device copy of a libgts result CSR as torch tensors (frees the handle)."""
    L = _lib.lib()
    try:
        nq, tot = C.c_int64(), C.c_int64()
        _lib.check(L.gts_result_info(h, C.byref(nq), C.byref(tot), None, None))
        off = torch.empty(nq.value + 1, dtype=torch.int64, device=device)
        ids = torch.empty(max(tot.value, 1), dtype=torch.int64, device=device)
        dis = torch.empty(max(tot.value, 1), dtype=torch.float64, device=device)
        _lib.check(L.gts_result_copy(h, C.cast(off.data_ptr(), _lib._i64p), C.cast(ids.data_ptr(), _lib._i64p),
                                     C.cast(dis.data_ptr(), _lib._f64p), None, None, C.c_void_p(stream)))
        return off, ids[:tot.value], dis[:tot.value]
    finally:
        L.gts_result_free(h)


class ShardSearcher:
    """One rank's shard index under torch.distributed: a device-resident
    query batch, the kNN probe, the bounded kNN search and range search, with
    answers as device tensors for `ShardExchange`."""

    def __init__(self, index_handle, device, memory_units=0, pruning=True, stream=None):
        self.ix = index_handle
        self.device = device
        self.memory_units = int(memory_units)
        self.pruning = pruning
        self.stream = stream if stream is not None else torch.cuda.current_stream(device).cuda_stream
        self.q = None
        self.nq = 0

    def upload(self, qb):
        """qb: a GtsQueryBatch (host payloads) -> device-resident batch."""
        self.free()
        q = C.c_void_p()
        _lib.check(_lib.lib().gts_queries_upload(self.ix, C.byref(qb), C.c_void_p(self.stream), C.byref(q)))
        self.q, self.nq = q, int(qb.nq)

    def free(self):
        if self.q:
            _lib.lib().gts_queries_free(self.q)
            self.q = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def probe(self, ks):
        """Per-query probe radius (float32 [nq] on the device)."""
        r = torch.empty(max(self.nq, 1), dtype=torch.float32, device=self.device)
        _lib.check(_lib.lib().gts_knn_probe(self.ix, self.q, _lib.ptr(ks, _lib._i64p), C.c_void_p(self.stream),
                                            C.c_void_p(r.data_ptr())))
        return r[:self.nq]

    def range(self, radii):
        h = C.c_void_p()
        _lib.check(_lib.lib().gts_range_batch(self.ix, self.q, _lib.ptr(radii, _lib._f64p), self.memory_units,
                                              int(self.pruning), C.c_void_p(self.stream), C.byref(h)))
        return result_tensors(h, self.device, self.stream)

    def knn(self, ks, radius=None):
        h = C.c_void_p()
        flags = _lib.FLAG_PRUNING if self.pruning else 0
        _lib.check(_lib.lib().gts_knn_batch_bounded(
            self.ix, self.q, _lib.ptr(ks, _lib._i64p), C.c_void_p(radius.data_ptr()) if radius is not None else None,
            self.memory_units, flags, C.c_void_p(self.stream), C.byref(h)))
        return result_tensors(h, self.device, self.stream)


def sharded_step(searcher, exchange, radii, ks, ks_dev, modes=(0, 1)):
    """One replicated batch over a sharded collection: range answers (mode 0)
    and kNN answers (mode 1: probe -> MIN bound -> bounded search), each
    merged on its owner.  Returns one (offsets, ids, dis) per mode for this
    rank's query slice."""
    out = []
    for m in modes:
        if m == 0:
            out.append(exchange.merge_range(*searcher.range(radii)))
        else:
            r = exchange.knn_bound(searcher.probe(ks))
            out.append(exchange.merge_knn(*searcher.knn(ks, r), ks_dev))
    return tuple(out)


# ---------------------------------------------------------------------------
# one process, several shard indexes (one per device in `devices`)
# ---------------------------------------------------------------------------

class ShardedIndex:
    """A collection split into contiguous id ranges, one GTS tree per shard,
    queried through one object with BatchSearcher's API and semantics.

    devices: the GPUs of the index (shard i lives on devices[i % len]);
    shards: number of shards (default len(devices))."""

    def __init__(self, dataset, config=None, devices=(0,), shards=None, memory_units=None, pruning=True):
        self.config = config or TreeConfig()
        self.dataset = dataset
        self.devices = list(devices)
        S = int(shards or len(self.devices))
        if S < 1:
            raise ValueError("need at least one shard")
        n = dataset.n
        self.bounds = [n * i // S for i in range(S + 1)]
        self.capacity = DEVICE_MEMORY_UNITS if memory_units is None else int(memory_units)
        self.pruning = pruning
        self.trees = []
        self._keep = []
        handles = []
        for i in range(S):
            rows = np.arange(self.bounds[i], self.bounds[i + 1])
            sub = dataset.subset_rows(rows)
            tree = build_tree(sub, self.config)
            if tree.n > 0 and self.capacity != DEVICE_MEMORY_UNITS and self.capacity < tree.nc:
                raise BudgetError(f"memory_units {self.capacity} below fan-out {tree.nc}")
            self.trees.append(tree)
            if tree.levels == 0:
                continue
            handles.append(tree.device_index(self.devices[i % len(self.devices)]).h)
        self._searcher = BatchSearcher(self.trees[0], memory_units=self.capacity, pruning=pruning,
                                       device=self.devices[0]) if self.trees else None
        self._m = None
        if handles:
            arr = (C.c_void_p * len(handles))(*handles)
            m = C.c_void_p()
            _lib.check(_lib.lib().gts_multi_create(len(handles), arr, C.byref(m)))
            self._m = m

    def __del__(self):
        try:
            if self._m:
                _lib.lib().gts_multi_destroy(self._m)
                self._m = None
        except Exception:
            pass

    @property
    def n(self):
        return self.dataset.n

    def range_batch(self, payloads, radii):
        res = self.range_batch_array(payloads, radii)
        return res.answers(), res.stats

    def knn_batch(self, payloads, ks):
        res = self.knn_batch_array(payloads, ks)
        return res.answers(), res.stats

    def range_batch_array(self, payloads, radii):
        nq = len(payloads)
        radii = np.ascontiguousarray(BatchSearcher._broadcast(radii, nq, "radius"))
        if np.any(radii < 0):
            raise ValueError("radius must be >= 0")
        return self._run(RANGE, payloads, radii, None)

    def knn_batch_array(self, payloads, ks):
        nq = len(payloads)
        ks = np.ascontiguousarray(BatchSearcher._broadcast(ks, nq, "k").astype(np.int64))
        if np.any(ks < 1):
            raise ValueError("k must be >= 1")
        return self._run(KNN, payloads, None, ks)

    def _run(self, mode, payloads, radii, ks):
        from .search import _fetch
        nq = len(payloads)
        if nq == 0 or self._m is None:
            if nq:
                self.dataset.prepare_batch(payloads)
            return CsrResult(np.zeros(nq + 1, dtype=np.int64), np.empty(0, np.int64), np.empty(0), SearchStats(nq))
        qb, keep = self._searcher._batch_struct(payloads)
        h = C.c_void_p()
        flags = _lib.FLAG_PRUNING if self.pruning else 0
        _lib.check(_lib.lib().gts_multi_batch_host(
            self._m, C.byref(qb), 0 if mode == RANGE else 1,
            _lib.ptr(radii, _lib._f64p) if radii is not None else None,
            _lib.ptr(ks, _lib._i64p) if ks is not None else None, max(self.capacity, 0), flags, C.byref(h)))
        return _fetch(h, nq)


__all__ = ["ShardedIndex", "ShardExchange", "ShardSearcher", "device_merge", "sharded_step"]
