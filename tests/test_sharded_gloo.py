"""Multi-shard exchange (the N>1 exchange step) on CPU with gloo, world size 2
and 3.

Each rank holds one shard of the dataset; its per-shard exact answers come
from the CPU oracle (the device search and the device merge kernel are
covered by tests/test_gpu_sharded.py).  `ShardExchange` partitions the
queries by owner, all-to-alls the answers and merges them; the merge is
injected here as a host restatement of k_merge_rank's contract, so what is
checked is the partitioning, the split sizes, the 16-byte packing and the
MIN bound all-reduce.  Every owner's slice must equal brute force over the
whole dataset.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT  # noqa: F401


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def host_merge(counts, ids, dis, ks):
    """k smallest (range: all) (distance, id) per query of S sorted lists."""
    S, nq = counts.shape
    c = counts.numpy()
    starts = np.concatenate([[0], np.cumsum(c.reshape(-1))])
    out_i, out_d, off = [], [], [0]
    for q in range(nq):
        segs = [(starts[s * nq + q], starts[s * nq + q + 1]) for s in range(S)]
        d = np.concatenate([dis.numpy()[a:b] for a, b in segs])
        i = np.concatenate([ids.numpy()[a:b] for a, b in segs])
        o = np.lexsort((i, d))
        if ks is not None:
            o = o[: int(ks[q])]
        out_i.append(i[o])
        out_d.append(d[o])
        off.append(off[-1] + o.size)
    return (torch.tensor(off, dtype=torch.int64), torch.from_numpy(np.concatenate(out_i).astype(np.int64)),
            torch.from_numpy(np.concatenate(out_d)))


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2404_00966_b200.sharded import ShardExchange
        rng = np.random.default_rng(0)
        n, nq = 3000, 41
        mat = np.round(rng.uniform(0, 10, size=(n, 3)))       # tie-heavy integer grid
        q = np.round(rng.uniform(0, 10, size=(nq, 3)))
        ids = np.arange(n, dtype=np.int64) * 3 + 7
        lo, hi = rank * n // world, (rank + 1) * n // world
        shard = O.Payloads(O.L1, vec=mat[lo:hi], ids=ids[lo:hi])
        qs = O.Payloads(O.L1, vec=q)
        ks = rng.integers(1, 30, nq)
        radii = rng.uniform(0, 4, nq)
        loc_k = O.brute(shard, qs, O.KNN, ks=ks)
        loc_r = O.brute(shard, qs, O.RANGE, radii=radii)
        ex = ShardExchange(nq, torch.device("cpu"), merge=host_merge)
        t = lambda r: (torch.from_numpy(r.offsets), torch.from_numpy(r.ids), torch.from_numpy(r.dis))
        ko, ki, kd = ex.merge_knn(*t(loc_k), torch.from_numpy(ks))
        ro, ri, rd = ex.merge_range(*t(loc_r))
        # the MIN bound exchange: every rank ends with the global minimum
        want_b = torch.tensor(rng.uniform(0, 1, nq).astype(np.float32))
        bound = want_b + rank
        ex.knn_bound(bound)
        qlo, qhi = ex.own
        full = O.Payloads(O.L1, vec=mat, ids=ids)
        sub = O.Payloads(O.L1, vec=q[qlo:qhi])
        wk = O.brute(full, sub, O.KNN, ks=ks[qlo:qhi])
        wr = O.brute(full, sub, O.RANGE, radii=radii[qlo:qhi])
        out[rank] = bool(np.array_equal(ko.numpy(), wk.offsets) and np.array_equal(ki.numpy(), wk.ids)
                         and np.array_equal(kd.numpy(), wk.dis) and np.array_equal(ro.numpy(), wr.offsets)
                         and np.array_equal(ri.numpy(), wr.ids) and np.array_equal(rd.numpy(), wr.dis)
                         and torch.equal(bound, want_b) and qhi - qlo == len(range(nq)[qlo:qhi]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_exchange_equals_brute_force(world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert dict(out) == {r: True for r in range(world)}
