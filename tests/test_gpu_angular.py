"""Angular metric on the device: fp32 cosine
screen with a rigorous arccos error band, exact float64 recheck in numpy's
order (pairwise dot and norms, arccos, zero-vector and identical-vector
rules).  Parity at the north star's float tolerance, applied at 1e-12
relative / 1e-14 absolute (see tests/test_angular.py for why angular cannot
be bit-exact with numpy's SIMD arccos)."""

import os

import numpy as np
import pytest

import paper_2404_00966_b200 as P
from conftest import load_golden
from oracle import oracle as O

pytestmark = pytest.mark.gpu
ANG = 3
REL, ABS = 1e-12, 1e-14


def csr(answers):
    return (np.array([a[0].size for a in answers]),
            np.concatenate([a[0] for a in answers]) if answers else np.empty(0, np.int64),
            np.concatenate([a[1] for a in answers]) if answers else np.empty(0))


def close(a, b):
    return a.shape == b.shape and np.allclose(a, b, rtol=REL, atol=ABS)


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def test_angular_pairs_match_reference():
    m = np.load(os.path.join(os.path.dirname(__file__), "golden", "metrics_angular.npz"))
    for k in m.files:
        if k.endswith("_d"):
            base = k[:-2]
            got = P.pair_distances(P.ANGULAR, m[base + "_a"], m[base + "_b"])
            assert close(got, m[k]), k
            exact = (m[k] == 0.0) | (m[k] == np.pi)
            assert np.array_equal(got[exact], m[k][exact]), k


def test_angular_golden_tree():
    g = load_golden("angular_16d")
    ds = P.Dataset.from_vectors(g["data_vec"], P.ANGULAR, ids=g["ids"])
    tree = P.build(ds, P.TreeConfig(int(g["nc"]), int(g["seed"])))
    queries = [g["query_vec"][i] for i in range(g["query_vec"].shape[0])]
    eng = P.BatchSearcher(tree)
    ans, st = eng.range_batch(queries, g["radii"])
    c, i, d = csr(ans)
    assert np.array_equal(c, g["range_wide_counts"]) and np.array_equal(i, g["range_wide_ids"])
    assert close(d, g["range_wide_dis"])
    assert np.all(st.verified >= g["range_wide_verified"])      # fp32 slack only adds work
    ans, _ = eng.knn_batch(queries, g["ks"])
    c, i, d = csr(ans)
    assert np.array_equal(c, g["knn_wide_counts"]) and np.array_equal(i, g["knn_wide_ids"])
    assert close(d, g["knn_wide_dis"])
    # tombstones
    tree.tombstone[:] = g["tombstone"]
    ans, _ = P.BatchSearcher(tree).range_batch(queries, g["radii"])
    c, i, d = csr(ans)
    assert np.array_equal(i, g["dead_range_wide_ids"]) and close(d, g["dead_range_wide_dis"])


@pytest.mark.parametrize("dim,n", [(3, 20000), (32, 20000), (100, 8000)])
def test_angular_vs_oracle(dim, n):
    rng = np.random.default_rng(dim)
    mat = f32(P.generate_clustered(n, dim, 40, seed=dim, spread=0.1) - 0.5)
    mat[:3] = 0.0                                      # zero vectors
    mat[3:10] = mat[500:507]                           # duplicates
    ds = P.Dataset.from_vectors(mat, P.ANGULAR)
    tree = P.build(ds, P.TreeConfig(12, 1))
    nq = 60
    q = np.concatenate([mat[rng.integers(0, n, nq // 2)],
                        f32(mat[rng.integers(0, n, nq - nq // 2 - 1)] * 1.7 + rng.normal(0, 0.02, (nq - nq // 2 - 1, dim))),
                        np.zeros((1, dim))])
    q = f32(q)
    radii = rng.uniform(0.0, 0.5, nq)
    ks = rng.integers(1, 40, nq)
    od, oq = O.Payloads(ANG, vec=mat), O.Payloads(ANG, vec=q)
    eng = P.BatchSearcher(tree)
    ans, _ = eng.range_batch(list(q), radii)
    c, i, d = csr(ans)
    want = O.brute(od, oq, O.RANGE, radii=radii, threads=8)
    assert np.array_equal(c, want.counts) and np.array_equal(i, want.ids)
    assert close(d, want.dis)
    ans, _ = eng.knn_batch(list(q), ks)
    c, i, d = csr(ans)
    want = O.brute(od, oq, O.KNN, ks=ks, threads=8)
    assert np.array_equal(c, want.counts) and np.array_equal(i, want.ids)
    assert close(d, want.dis)


def test_angular_streaming_index():
    rng = np.random.default_rng(3)
    dim = 8
    mat = f32(rng.normal(size=(3000, dim)))
    si = P.StreamingIndex(P.Dataset.from_vectors(mat, P.ANGULAR), P.TreeConfig(8, 0), cache_capacity=64)
    live = {i: mat[i] for i in range(3000)}
    nid = 3000
    for step in range(4):
        for oid in rng.choice(sorted(live), 40, replace=False):
            si.delete(int(oid))
            del live[int(oid)]
        for _ in range(30):
            v = f32(rng.normal(size=dim))
            si.insert(nid, v)
            live[nid] = v
            nid += 1
        ids = np.array(sorted(live), dtype=np.int64)
        od = O.Payloads(ANG, vec=np.array([live[i] for i in ids]), ids=ids)
        q = f32(rng.normal(size=(12, dim)))
        oq = O.Payloads(ANG, vec=q)
        got, _ = si.query_range(list(q), 0.4)
        want = O.brute(od, oq, O.RANGE, radii=np.full(12, 0.4))
        c, i, d = csr(got)
        assert np.array_equal(i, want.ids) and close(d, want.dis)
        got, _ = si.query_knn(list(q), 6)
        want = O.brute(od, oq, O.KNN, ks=np.full(12, 6))
        c, i, d = csr(got)
        assert np.array_equal(i, want.ids) and close(d, want.dis)
