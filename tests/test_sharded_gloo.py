"""Multi-shard merge (the N>1 exchange step) on CPU with gloo, world size 2.

Each rank holds one shard of the dataset; per-shard exact answers come from
the CPU oracle (the device search is covered by the GPU tests); the merged
answers must equal brute force over the whole dataset.
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


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2404_00966_b200.sharded import ShardMerger
        rng = np.random.default_rng(0)
        n = 3000
        mat = np.round(rng.uniform(0, 10, size=(n, 3)))       # tie-heavy integer grid
        q = np.round(rng.uniform(0, 10, size=(40, 3)))
        ids = np.arange(n, dtype=np.int64)
        lo, hi = rank * n // world, (rank + 1) * n // world
        shard = O.Payloads(O.L1, vec=mat[lo:hi], ids=ids[lo:hi])
        qs = O.Payloads(O.L1, vec=q)
        ks = rng.integers(1, 30, 40)
        radii = rng.uniform(0, 4, 40)
        loc_k = O.brute(shard, qs, O.KNN, ks=ks)
        loc_r = O.brute(shard, qs, O.RANGE, radii=radii)
        m = ShardMerger(40, torch.device("cpu"))
        t = lambda r: (torch.from_numpy(r.offsets), torch.from_numpy(r.ids), torch.from_numpy(r.dis))
        ko, ki, kd = m.merge_knn(*t(loc_k), ks)
        ro, ri, rd = m.merge_range(*t(loc_r))
        if rank == 0:
            full = O.Payloads(O.L1, vec=mat, ids=ids)
            wk = O.brute(full, qs, O.KNN, ks=ks)
            wr = O.brute(full, qs, O.RANGE, radii=radii)
            out["ok"] = bool(np.array_equal(ko.numpy(), wk.offsets) and np.array_equal(ki.numpy(), wk.ids)
                             and np.array_equal(kd.numpy(), wk.dis) and np.array_equal(ro.numpy(), wr.offsets)
                             and np.array_equal(ri.numpy(), wr.ids) and np.array_equal(rd.numpy(), wr.dis))
    finally:
        dist.destroy_process_group()


def test_two_shard_merge_equals_brute_force():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out.get("ok") is True
