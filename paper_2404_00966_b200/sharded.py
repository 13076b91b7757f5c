"""Multi-GPU sharding: one GTS tree per GPU, query batch replicated, per-shard
answers merged (BASELINE.json north_star).

Exact search over a partition is the union of exact per-shard answers
(Def. 1/2), so the only exchange step is the merge:
  kNN   : every shard's top-k per query (padded to k) is all-gathered and the
          k smallest (distance, id) pairs of the union are kept;
  range : per-shard CSR hits are all-gathered and re-sorted by (distance, id)
          per query.
The merge runs on torch tensors with torch.distributed collectives (NCCL
over NVLink on GPUs; gloo on CPU in the tests).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

_ID_PAD = np.iinfo(np.int64).max


def _lex_sort(q, d, ids):
    """Permutation ordering rows by (q, d, id) via three stable sorts."""
    p = torch.argsort(ids, stable=True)
    p = p[torch.argsort(d[p], stable=True)]
    p = p[torch.argsort(q[p], stable=True)]
    return p


def merge_knn_dense(d_all, id_all, ks):
    """d_all/id_all: [S, nq, kmax] (inf / ID_PAD padded).  Returns CSR
    (offsets, ids, dis) of the k smallest (d, id) per query."""
    S, nq, kmax = d_all.shape
    d = d_all.permute(1, 0, 2).reshape(nq, S * kmax)
    ids = id_all.permute(1, 0, 2).reshape(nq, S * kmax)
    q = torch.arange(nq, device=d.device).repeat_interleave(S * kmax)
    d, ids = d.reshape(-1), ids.reshape(-1)
    p = _lex_sort(q, d, ids)
    d, ids = d[p].reshape(nq, S * kmax), ids[p].reshape(nq, S * kmax)
    ks = torch.as_tensor(ks, device=d.device).reshape(-1, 1)
    rank = torch.arange(S * kmax, device=d.device).reshape(1, -1)
    keep = (rank < ks) & torch.isfinite(d)
    counts = keep.sum(dim=1)
    offsets = torch.zeros(nq + 1, dtype=torch.int64, device=d.device)
    offsets[1:] = torch.cumsum(counts, 0)
    return offsets, ids[keep], d[keep]


def merge_range_flat(q_all, d_all, id_all):
    """Flat (query, distance, id) hits from every shard -> CSR sorted by (d, id)."""
    p = _lex_sort(q_all, d_all, id_all)
    return p


def csr_to_dense(offsets, ids, dis, kmax):
    nq = offsets.numel() - 1
    counts = offsets[1:] - offsets[:-1]
    D = torch.full((nq, kmax), float("inf"), dtype=torch.float64, device=dis.device)
    I = torch.full((nq, kmax), _ID_PAD, dtype=torch.int64, device=ids.device)
    if ids.numel():
        q = torch.repeat_interleave(torch.arange(nq, device=ids.device), counts)
        r = torch.arange(ids.numel(), device=ids.device) - offsets[:-1][q]
        D[q, r] = dis
        I[q, r] = ids
    return D, I


class ShardMerger:
    """All-gather + merge of per-shard results for one query batch."""

    def __init__(self, nq, device, group=None):
        self.nq = nq
        self.device = device
        self.group = group

    def _world(self):
        return dist.get_world_size(self.group) if dist.is_initialized() else 1

    def merge_knn(self, offsets, ids, dis, ks):
        ks_t = torch.as_tensor(np.asarray(ks), device=self.device)
        kmax = int(ks_t.max().item()) if ks_t.numel() else 1
        D, I = csr_to_dense(offsets, ids, dis, kmax)
        S = self._world()
        if S > 1:
            Ds = [torch.empty_like(D) for _ in range(S)]
            Is = [torch.empty_like(I) for _ in range(S)]
            dist.all_gather(Ds, D, group=self.group)
            dist.all_gather(Is, I, group=self.group)
            D, I = torch.stack(Ds), torch.stack(Is)
        else:
            D, I = D[None], I[None]
        return merge_knn_dense(D, I, ks_t)

    def merge_range(self, offsets, ids, dis):
        nq = offsets.numel() - 1
        counts = offsets[1:] - offsets[:-1]
        q = torch.repeat_interleave(torch.arange(nq, device=ids.device), counts)
        S = self._world()
        if S > 1:
            n = torch.tensor([ids.numel()], device=ids.device)
            ns = [torch.empty_like(n) for _ in range(S)]
            dist.all_gather(ns, n, group=self.group)
            m = int(max(x.item() for x in ns))
            def pad(t, v):
                out = torch.full((m,), v, dtype=t.dtype, device=t.device)
                out[: t.numel()] = t
                return out
            parts = []
            for t, v in ((q, nq), (dis, float("inf")), (ids, _ID_PAD)):
                lst = [torch.empty(m, dtype=t.dtype, device=t.device) for _ in range(S)]
                dist.all_gather(lst, pad(t, v), group=self.group)
                parts.append(torch.cat([x[: int(c.item())] for x, c in zip(lst, ns)]))
            q, dis, ids = parts
        p = _lex_sort(q, dis, ids)
        q, dis, ids = q[p], dis[p], ids[p]
        counts = torch.bincount(q, minlength=nq)
        offsets = torch.zeros(nq + 1, dtype=torch.int64, device=ids.device)
        offsets[1:] = torch.cumsum(counts, 0)
        return offsets, ids, dis

    # -- bench / API glue: copy a libgts result (device CSR) into tensors ----
    def tensors_of(self, eng, h, stream):
        from . import _lib
        nq, tot = eng.info(h)
        off = torch.empty(nq + 1, dtype=torch.int64, device=self.device)
        ids = torch.empty(max(tot, 1), dtype=torch.int64, device=self.device)
        dis = torch.empty(max(tot, 1), dtype=torch.float64, device=self.device)
        _lib.check(eng.L.gts_result_copy(h, C.cast(off.data_ptr(), _lib._i64p), C.cast(ids.data_ptr(), _lib._i64p),
                                         C.cast(dis.data_ptr(), _lib._f64p), None, None, C.c_void_p(stream)))
        return off, ids[:tot], dis[:tot]

    def merge_handles(self, eng, hs, ks, stream):
        r = self.merge_range(*self.tensors_of(eng, hs[0], stream))
        k = self.merge_knn(*self.tensors_of(eng, hs[1], stream), ks)
        return r, k
