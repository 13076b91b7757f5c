"""Sharded collections on the device: the merge kernel
(k_merge_rank), the one-process multi-shard handle (gts_multi_*), and the
per-rank path (probe -> MIN bound -> bounded kNN, owner all-to-all, device
merge) with two ranks sharing cuda:0 over gloo.  Every answer must equal the
oracle's brute force over the whole collection (oracle.py:19-36)."""

import os
import socket

import numpy as np
import pytest
import torch

import paper_2404_00966_b200 as P
from oracle import oracle as O
from paper_2404_00966_b200.sharded import ShardedIndex, device_merge
from test_sharded_gloo import host_merge

pytestmark = pytest.mark.gpu


def _csr(ans):
    off = np.zeros(len(ans) + 1, np.int64)
    np.cumsum([a[0].size for a in ans], out=off[1:])
    ids = np.concatenate([a[0] for a in ans]) if ans else np.zeros(0, np.int64)
    dis = np.concatenate([a[1] for a in ans]) if ans else np.zeros(0)
    return off, ids, dis


def _same(ans, want):
    off, ids, dis = _csr(ans)
    return np.array_equal(off, want.offsets) and np.array_equal(ids, want.ids) and np.array_equal(dis, want.dis)


@pytest.mark.parametrize("S", [1, 2, 5])
def test_device_merge_matches_host_merge(S):
    rng = np.random.default_rng(S)
    nq = 300
    counts = rng.integers(0, 40, size=(S, nq))
    counts[:, :7] = 0
    ids_all = rng.permutation(10**6)[: counts.sum()].astype(np.int64)
    parts_i, parts_d, k = [], [], 0
    for s in range(S):
        for q in range(nq):
            c = int(counts[s, q])
            d = np.round(rng.uniform(0, 5, c))   # many distance ties across sources
            i = ids_all[k:k + c]
            k += c
            o = np.lexsort((i, d))
            parts_i.append(i[o])
            parts_d.append(d[o])
    ids = np.concatenate(parts_i)
    dis = np.concatenate(parts_d)
    ks = rng.integers(1, 60, nq)
    dev = torch.device("cuda", 0)
    tc = torch.from_numpy(counts.astype(np.int64))
    for kk in (ks, None):
        got = device_merge(tc.to(dev), torch.from_numpy(ids).to(dev), torch.from_numpy(dis).to(dev),
                           None if kk is None else torch.from_numpy(kk).to(dev))
        want = host_merge(tc, torch.from_numpy(ids), torch.from_numpy(dis), kk)
        for g, w in zip(got, want):
            assert torch.equal(g.cpu(), w)


def _edit_data(n, seed):
    strs = P.generate_sequences(n, seed=seed, min_len=1, max_len=20, alphabet="abcdefgh")
    rng = np.random.default_rng(seed)
    q = [strs[int(i)] for i in rng.integers(0, n, 40)] + ["", "zzzz", "abcabcabc"]
    return P.Dataset.from_strings(strs, P.EDIT, ids=np.arange(n) * 2 + 1), q


@pytest.mark.parametrize("metric", ["edit", "l2", "l1"])
@pytest.mark.parametrize("shards", [2, 3])
def test_sharded_index_equals_brute_force(metric, shards):
    rng = np.random.default_rng(7)
    if metric == "edit":
        ds, q = _edit_data(6000, 3)
        od = O.Payloads.from_strings(ds.strings, ids=ds.ids)
        oq = O.Payloads.from_strings(q)
        radii = rng.integers(0, 4, len(q)).astype(float)
    else:
        D = 2 if metric == "l2" else 32
        mat = rng.uniform(0, 1, (8000, D)).astype(np.float32).astype(np.float64)
        code = P.L2 if metric == "l2" else P.L1
        ds = P.Dataset.from_vectors(mat, code)
        q = list(mat[rng.integers(0, 8000, 40)] + rng.normal(0, 0.01, (40, D)).astype(np.float32))
        od = O.Payloads(O.L2 if metric == "l2" else O.L1, vec=mat)
        oq = O.Payloads(od.metric, vec=np.asarray(q, dtype=np.float64))
        radii = rng.uniform(0.0, 0.1 if D == 2 else 1.5, len(q))
    ks = rng.integers(1, 40, len(q))
    ks[0] = 5000   # k above a whole shard: every shard returns all its live objects
    six = ShardedIndex(ds, P.TreeConfig(20, 0), devices=[0], shards=shards)
    ra, rs = six.range_batch(q, radii)
    ka, kst = six.knn_batch(q, ks)
    assert _same(ra, O.brute(od, oq, O.RANGE, radii=radii, threads=8))
    assert _same(ka, O.brute(od, oq, O.KNN, ks=ks, threads=8))
    assert rs.verified.sum() > 0


def test_knn_k_above_probe_cap_uses_finite_radius():
    """k > 8192 (the probe's candidate cap) on a float metric: the search
    starts from the root-radius bound instead of +inf and stays exact."""
    rng = np.random.default_rng(1)
    mat = rng.uniform(0, 1, (40000, 2)).astype(np.float32).astype(np.float64)
    tree = P.build(P.Dataset.from_vectors(mat, P.L2), P.TreeConfig(20, 0))
    q = list(mat[:6])
    ks = np.array([9000, 12000, 10, 8193, 20000, 1])
    ans, _ = P.BatchSearcher(tree).knn_batch(q, ks)
    want = O.brute(O.Payloads(O.L2, vec=mat), O.Payloads(O.L2, vec=np.asarray(q)), O.KNN, ks=ks, threads=8)
    assert _same(ans, want)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_worker(rank, world, port, out):
    import ctypes as C
    import torch.distributed as dist
    from paper_2404_00966_b200 import _lib
    from paper_2404_00966_b200.sharded import ShardExchange, ShardSearcher, sharded_step
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        ds, q = _edit_data(9000, 11)
        n = ds.n
        lo, hi = rank * n // world, (rank + 1) * n // world
        shard = ds.subset_rows(np.arange(lo, hi))
        tree = P.build(shard, P.TreeConfig(20, 0))
        h = tree.device_index(0).h
        searcher = P.BatchSearcher(tree)
        qb, keep = searcher._batch_struct(q)
        ss = ShardSearcher(h, dev)
        ss.upload(qb)
        nq = len(q)
        rng = np.random.default_rng(2)
        radii = rng.integers(0, 4, nq).astype(np.float64)
        ks = rng.integers(1, 30, nq).astype(np.int64)
        ex = ShardExchange(nq, dev)
        (ro, ri, rd), (ko, ki, kd) = sharded_step(ss, ex, radii, ks, torch.from_numpy(ks).to(dev))
        torch.cuda.synchronize()
        qlo, qhi = ex.own
        od = O.Payloads.from_strings(ds.strings, ids=ds.ids)
        oq = O.Payloads.from_strings(q[qlo:qhi])
        wr = O.brute(od, oq, O.RANGE, radii=radii[qlo:qhi], threads=4)
        wk = O.brute(od, oq, O.KNN, ks=ks[qlo:qhi], threads=4)
        ok = all(np.array_equal(a.cpu().numpy(), b) for a, b in
                 ((ro, wr.offsets), (ri, wr.ids), (rd, wr.dis), (ko, wk.offsets), (ki, wk.ids), (kd, wk.dis)))
        out[rank] = ok
        ss.free()
    finally:
        dist.destroy_process_group()


def test_two_ranks_device_answers_exchange_and_merge():
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_rank_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert dict(out) == {0: True, 1: True}
