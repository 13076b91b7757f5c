"""Device-resident collections: the Philox generator is
counter-based (any slice equals the same rows of the whole), and an index
created over device float32 payloads (gts_build_tree_device_f32 +
gts_index_create_f32dev) answers exactly like the host-built index over the
same values and like the oracle's brute force."""

import ctypes as C

import numpy as np
import pytest
import torch

import paper_2404_00966_b200 as P
from oracle import oracle as O
from paper_2404_00966_b200 import _lib
from paper_2404_00966_b200.search import _fetch
from paper_2404_00966_b200.tree import node_count_for

pytestmark = pytest.mark.gpu


def gen(n_total, D, first, count, qseed=0, clusters=50, spread=0.05, noise=0.01):
    x = torch.empty((count, D), dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().gts_generate_clustered(12, n_total, D, clusters, spread, first, count, qseed, noise,
                                                 C.c_void_p(x.data_ptr()), None))
    torch.cuda.synchronize()
    return x


def test_generator_is_counter_based():
    whole = gen(10007, 32, 0, 10007).cpu()
    parts = torch.cat([gen(10007, 32, a, min(10007, a + 3001) - a).cpu() for a in range(0, 10007, 3001)])
    assert torch.equal(whole, parts)
    q1, q2 = gen(10007, 32, 0, 500, qseed=13).cpu(), gen(10007, 32, 100, 50, qseed=13).cpu()
    assert torch.equal(q1[100:150], q2)
    assert torch.isfinite(whole).all() and 0.3 < float(whole.mean()) < 0.7
    assert not torch.equal(gen(10007, 5, 0, 10, qseed=0).cpu(), gen(10007, 5, 0, 10, qseed=13).cpu())


def device_index(x, metric_code, ids):
    n, D = x.shape
    ds = P.Dataset.from_vectors(x.double().cpu().numpy(), P.L1 if metric_code == 1 else P.L2, ids=ids)
    tree = P.FlatPivotTree(P.TreeConfig(20, 0), ds)
    tree.max_h, tree.split_rounds = P.tree_height(n, 20)
    tree.levels = tree.split_rounds + 1
    tree._alloc_nodes(node_count_for(tree.levels, 20))
    t = tree._c_tree()
    root = int(np.random.default_rng(0).integers(0, n))
    _lib.check(_lib.lib().gts_build_tree_device_f32(metric_code, n, D, C.c_void_p(x.data_ptr()),
                                                    _lib.ptr(ds.ids, _lib._i64p), root, 0, C.byref(t)))
    h = C.c_void_p()
    _lib.check(_lib.lib().gts_index_create_f32dev(C.byref(t), metric_code, D, C.c_void_p(x.data_ptr()),
                                                  _lib.ptr(ds.ids, _lib._i64p), 0, C.byref(h)))
    return ds, tree, h


def run(h, q, mode, code, radii=None, ks=None):
    nq, D = q.shape
    qb = _lib.GtsQueryBatch(code, nq, D, _lib.ptr(q, _lib._f64p), None, None)
    r = C.c_void_p()
    _lib.check(_lib.lib().gts_batch_host(h, C.byref(qb), mode,
                                         _lib.ptr(radii, _lib._f64p) if radii is not None else None,
                                         _lib.ptr(ks, _lib._i64p) if ks is not None else None, 0,
                                         _lib.FLAG_PRUNING, None, C.byref(r)))
    return _fetch(r, nq)


@pytest.mark.parametrize("metric_code,D", [(1, 32), (2, 64), (2, 20)])
def test_device_payload_index_matches_host_index_and_brute(metric_code, D):
    n = 120000
    x = gen(n, D, 0, n, clusters=300)
    ids = np.arange(n, dtype=np.int64) * 2 + 5
    ds, tree, h = device_index(x, metric_code, ids)
    try:
        q = gen(n, D, 0, 96, qseed=13, clusters=300).double().cpu().numpy()
        host_tree = P.build(ds, P.TreeConfig(20, 0))
        for f in ("pivot_id", "pivot_row", "min_dis", "max_dis", "pos", "size", "rows", "dis"):
            assert np.array_equal(getattr(host_tree, f), getattr(tree, f)), f
        radii = np.full(96, 0.3 if metric_code == 1 else 0.08)
        ks = np.full(96, 100, dtype=np.int64)
        got_r, got_k = run(h, q, 0, metric_code, radii=radii), run(h, q, 1, metric_code, ks=ks)
        eng = P.BatchSearcher(host_tree)
        want_r, want_k = eng.range_batch_array(list(q), radii), eng.knn_batch_array(list(q), ks)
        for g, w_ in ((got_r, want_r), (got_k, want_k)):
            assert np.array_equal(g.offsets, w_.offsets) and np.array_equal(g.ids, w_.ids)
            assert np.array_equal(g.dis, w_.dis)
        od = O.Payloads(O.L1 if metric_code == 1 else O.L2, vec=ds.mat, ids=ids)
        oq = O.Payloads(od.metric, vec=q)
        b = O.brute(od, oq, O.KNN, ks=ks, threads=8)
        assert np.array_equal(got_k.ids, b.ids) and np.array_equal(got_k.dis, b.dis)
    finally:
        _lib.lib().gts_index_destroy(h)
