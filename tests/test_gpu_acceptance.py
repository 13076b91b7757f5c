"""The reference's acceptance gates that exercise the search path, run
through this package's drop-in API on the device (test_acceptance.py):
#1 range exactness on every metric kind x six quantile radii (111-142),
#2 kNN exactness over k in {1..32} (148-183), #5 512-query batches inside a
1000-row budget with size_limits {1: 25, 2: 50} (245-269), #6 a 5,000-op
interleaved update stream at cache capacities 1 / 64 / 512 (275-331),
#10 pruning skips at least half the leaf work on clustered data (433-460).
The checker is the oracle's brute force (oracle/ -- the reference's
oracle.py restated), never the product."""

import re

import numpy as np
import pytest

import paper_2404_00966_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu

RADIUS_SETTINGS = (1, 2, 4, 8, 16, 32)   # selectivity dial, 0.01 % steps
K_SETTINGS = (1, 2, 4, 8, 16, 32)


def stdlib_words(limit=5000):
    """Real English-ish words from stdlib docstrings (no files, no network)."""
    import collections, email, html, http, json, logging, os, pathlib, string, textwrap, typing, unittest, urllib
    words = set()
    for mod in (collections, email, html, http, json, logging, os, pathlib, string, textwrap, typing, unittest,
                urllib, re, np):
        for name in dir(mod):
            doc = getattr(getattr(mod, name, None), "__doc__", None) or ""
            if not isinstance(doc, str):   # e.g. a slot's member_descriptor
                continue
            for tok in re.findall(r"[a-z]{2,14}", doc.lower()):
                if re.search(r"[aeiouy]", tok) and not re.search(r"(.)\1\1", tok):
                    words.add(tok)
    return sorted(words)[:limit]


def dataset(kind, n=5000):
    if kind == "l1":
        return P.Dataset.from_vectors(np.round(P.generate_uniform(n, 4, seed=11) * 50), P.L1)
    if kind == "l2":
        return P.Dataset.from_vectors(P.generate_uniform(n, 2, seed=12), P.L2)
    if kind == "angular":
        return P.Dataset.from_vectors(P.generate_uniform(n, 3, seed=13) - 0.5, P.ANGULAR)
    if kind == "edit-synthetic":
        return P.Dataset.from_strings(P.generate_sequences(n, seed=14), P.EDIT)
    words = stdlib_words(n)
    assert len(words) >= 2000
    return P.Dataset.from_strings(words, P.EDIT)


def oracle_of(ds):
    if ds.metric == P.EDIT:
        return O.Payloads.from_strings(ds.strings, ids=ds.ids)
    return O.Payloads({P.L1: O.L1, P.L2: O.L2, P.ANGULAR: 3}[ds.metric], vec=ds.mat, ids=ds.ids)


def oq_of(ds, queries):
    if ds.metric == P.EDIT:
        return O.Payloads.from_strings(queries)
    return O.Payloads({P.L1: O.L1, P.L2: O.L2, P.ANGULAR: 3}[ds.metric], vec=np.array(queries))


def quantile_radii(ds, seed=0, samples=200_000):
    rng = np.random.default_rng(seed)
    a, b = rng.integers(0, ds.n, samples), rng.integers(0, ds.n, samples)
    keep = a != b
    pa = [ds.payload(int(i)) for i in a[keep]]
    pb = [ds.payload(int(i)) for i in b[keep]]
    d = P.pair_distances(ds.metric, pa, pb)
    floor = float(d[d > 0].min())
    return [max(float(np.quantile(d, v * 1e-4)), floor) for v in RADIUS_SETTINGS]


def queries_for(ds, nq, rng):
    if ds.metric != P.EDIT:
        mat = ds.mat
        members = [mat[int(i)].copy() for i in rng.integers(0, ds.n, nq // 2)]
        lo, hi = mat.min(axis=0), mat.max(axis=0)
        return members + [rng.uniform(lo, hi) for _ in range(nq - nq // 2)]
    strs = ds.strings
    alpha = sorted({c for s in strs[:200] for c in s})
    out = [strs[int(i)] for i in rng.integers(0, ds.n, nq // 2)]
    for i in rng.integers(0, ds.n, nq - nq // 2):
        s = list(strs[int(i)])
        for _ in range(int(rng.integers(1, 3))):
            c = alpha[int(rng.integers(0, len(alpha)))]
            if s and rng.integers(0, 2):
                s[int(rng.integers(0, len(s)))] = c
            else:
                s.insert(int(rng.integers(0, len(s) + 1)), c)
        out.append("".join(s))
    return out


def same(got, want, metric):
    if metric == P.ANGULAR:   # numpy's arccos is not libm's (tests/test_angular.py)
        return np.array_equal(got[0], want[0]) and np.allclose(got[1], want[1], rtol=1e-12, atol=1e-14)
    return np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


@pytest.mark.parametrize("kind,nq", [("l1", 1000), ("l2", 1000), ("angular", 1000), ("edit-synthetic", 500),
                                     ("edit-words", 500)])
def test_gate1_range_exact_every_metric(kind, nq):
    ds = dataset(kind)
    eng = P.BatchSearcher(P.build(ds, P.TreeConfig(20, 0)))
    rng = np.random.default_rng(100)
    q = queries_for(ds, nq, rng)
    menu = quantile_radii(ds)
    radii = np.array([menu[i % 6] for i in range(nq)])
    got, _ = eng.range_batch(q, radii)
    want = O.brute(oracle_of(ds), oq_of(ds, q), O.RANGE, radii=radii, threads=8).answers()
    assert all(same(g, w, ds.metric) for g, w in zip(got, want))
    assert sum(g[0].size > 0 for g in got) > 0


@pytest.mark.parametrize("kind", ["edit-synthetic", "l2"])
def test_gate2_knn_exact_k_grid(kind):
    ds = dataset(kind)
    eng = P.BatchSearcher(P.build(ds, P.TreeConfig(20, 0)))
    q = queries_for(ds, 1000, np.random.default_rng(200))
    ks = np.array([K_SETTINGS[i % 6] for i in range(1000)])
    got, _ = eng.knn_batch(q, ks)
    want = O.brute(oracle_of(ds), oq_of(ds, q), O.KNN, ks=ks, threads=8).answers()
    for (ids, d), (wi, wd), k in zip(got, want, ks):
        assert ids.size == k and len(set(ids.tolist())) == k and np.all(d[:-1] <= d[1:])
        assert d.tolist() == wd.tolist() and ids.tolist() == wi.tolist()


def test_gate5_budget_512_batch():
    cap = 1000
    ds = P.Dataset.from_vectors(P.generate_uniform(10**5, 2, seed=5), P.L2)
    tree = P.build(ds, P.TreeConfig(20, 0))
    assert tree.split_rounds == 2
    eng = P.BatchSearcher(tree, memory_units=cap)
    q = queries_for(ds, 512, np.random.default_rng(500))
    r = quantile_radii(ds)[3]
    got, st = eng.range_batch(q, r)
    assert st.peak_units <= cap
    assert st.size_limits == {1: 25, 2: 50}
    want = O.brute(oracle_of(ds), oq_of(ds, q), O.RANGE, radii=np.full(512, r), threads=8).answers()
    assert all(same(g, w, P.L2) for g, w in zip(got, want))
    kg, kst = eng.knn_batch(q, 8)
    assert kst.peak_units <= cap
    kw = O.brute(oracle_of(ds), oq_of(ds, q), O.KNN, ks=np.full(512, 8), threads=8).answers()
    assert all(same(g, w, P.L2) for g, w in zip(kg, kw))


@pytest.mark.parametrize("cap", [1, 64, 512])
def test_gate6_update_stream(cap):
    ops = 5000 // 3
    mat = P.generate_uniform(2000, 2, seed=cap)
    si = P.StreamingIndex(P.Dataset.from_vectors(mat, P.L2), P.TreeConfig(20, 0), cache_capacity=cap)
    tracked = {i: mat[i] for i in range(2000)}
    rng = np.random.default_rng(cap + 1)
    next_id, freed, mirror, rebuilds = 2000, [], set(), 0
    for _ in range(ops):
        roll = rng.uniform()
        if roll < 0.35:
            if freed and rng.integers(0, 2):
                obj = freed.pop(int(rng.integers(0, len(freed))))
            else:
                obj, next_id = next_id, next_id + 1
            p = rng.uniform(0, 1, 2)
            si.insert(obj, p)
            tracked[obj] = p
            mirror.add(obj)
            if len(mirror) > cap:
                mirror.clear()
                rebuilds += 1
        elif roll < 0.70 and tracked:
            obj = int(rng.choice(sorted(tracked)))
            si.delete(obj)
            del tracked[obj]
            freed.append(obj)
            mirror.discard(obj)
        else:
            ids = np.array(sorted(tracked), dtype=np.int64)
            od = O.Payloads(O.L2, vec=np.array([tracked[i] for i in ids]), ids=ids)
            q = rng.uniform(0, 1, 2)
            oq = O.Payloads(O.L2, vec=q[None])
            g, _ = si.query_range([q], 0.05)
            assert same(g[0], O.brute(od, oq, O.RANGE, radii=np.array([0.05])).answers()[0], P.L2)
            gk, _ = si.query_knn([q], 5)
            assert same(gk[0], O.brute(od, oq, O.KNN, ks=np.array([5])).answers()[0], P.L2)
    assert si.rebuild_count == rebuilds
    assert si.n_live == len(tracked)


def test_gate10_pruning_skips_half():
    mat = P.generate_clustered(10**5, 2, clusters=10, seed=10)
    ds = P.Dataset.from_vectors(mat, P.L2)
    tree = P.build(ds, P.TreeConfig(20, 0))
    # resolve_radius(ds, 8, "relative-diameter"): 8e-4 x a sampled diameter
    rng = np.random.default_rng(0)
    anchors = rng.integers(0, ds.n, 64)
    rows = rng.integers(0, ds.n, (64, 2000 // 64))
    diam = max(float(np.sqrt(((mat[rows[i]] - mat[a]) ** 2).sum(axis=1)).max()) for i, a in enumerate(anchors))
    radius = 8e-4 * diam
    q = [mat[int(i)].copy() for i in np.random.default_rng(1000).integers(0, ds.n, 64)]
    on, off = P.BatchSearcher(tree, pruning=True), P.BatchSearcher(tree, pruning=False)
    a_on, s_on = on.range_batch(q, radius)
    a_off, s_off = off.range_batch(q, radius)
    assert s_off.total_verified == 64 * ds.n
    assert 1.0 - s_on.total_verified / s_off.total_verified >= 0.5
    for x, y in zip(a_on, a_off):
        assert same(x, y, P.L2)
    want = O.brute(oracle_of(ds), oq_of(ds, q), O.RANGE, radii=np.full(64, radius), threads=8).answers()
    assert all(same(g, w, P.L2) for g, w in zip(a_on, want))
    k_on, _ = on.knn_batch(q[:16], 8)
    k_off, _ = off.knn_batch(q[:16], 8)
    kw = O.brute(oracle_of(ds), oq_of(ds, q[:16]), O.KNN, ks=np.full(16, 8), threads=8).answers()
    for x, y, w in zip(k_on, k_off, kw):
        assert same(x, y, P.L2) and same(x, w, P.L2)
