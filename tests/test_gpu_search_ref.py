"""The reference's batch-engine tests (tests/test_search.py:178-300) on the
device path: k beyond the collection, tie-heavy integer L1 grids, batch
equals sequential, runtime and budget never change answers, logged size
limits, pruning off, tombstones.  Expected answers come from the oracle's
brute force (oracle/, test infrastructure)."""

import numpy as np
import pytest

import paper_2404_00966_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def make_index(n, metric=P.L2, nc=4, seed=0, dim=2):
    """Same data as the reference helper (test_search.py:103-114)."""
    if metric == P.EDIT:
        payloads = P.generate_sequences(n, seed=seed)
        ds = P.Dataset.from_strings(payloads, metric)
        od = O.Payloads.from_strings(payloads)
    else:
        mat = P.generate_uniform(n, dim, seed=seed)
        if metric == P.L1:
            mat = np.round(mat * 8)   # integer grid: heavy ties
        ds = P.Dataset.from_vectors(mat, metric)
        payloads = [mat[i] for i in range(n)]
        od = O.Payloads({P.L1: 1, P.L2: 2}[metric], vec=mat)
    return P.build(ds, P.TreeConfig(node_capacity=nc, seed=seed)), ds, payloads, od


def oq_of(metric, queries):
    if metric == P.EDIT:
        return O.Payloads.from_strings(queries)
    return O.Payloads({P.L1: 1, P.L2: 2}[metric], vec=np.array(queries))


def pairs(answers):
    return [(ids.tolist(), dis.tolist()) for ids, dis in answers]


def assert_matches(answers, want):
    off = np.concatenate([[0], np.cumsum([a[0].size for a in answers])])
    assert np.array_equal(off, want.offsets)
    assert np.array_equal(np.concatenate([a[0] for a in answers]), want.ids)
    assert np.array_equal(np.concatenate([a[1] for a in answers]), want.dis)


@pytest.mark.parametrize("metric", [P.L2, P.L1, P.EDIT])
def test_knn_k_larger_than_collection(metric):
    tree, _, payloads, _ = make_index(10, metric=metric)
    answers, _ = P.BatchSearcher(tree).knn_batch([payloads[0]], 25)
    assert answers[0][0].size == 10
    assert answers[0][1].tolist() == sorted(answers[0][1].tolist())


def test_knn_tie_heavy_kth_distance_multiset():
    rng = np.random.default_rng(31)
    tree, _, payloads, od = make_index(240, metric=P.L1, nc=4, seed=3)
    eng = P.BatchSearcher(tree)
    queries = [payloads[int(i)] for i in rng.integers(0, 240, 16)]
    for k in (1, 3, 7, 16):
        answers, _ = eng.knn_batch(queries, k)
        assert_matches(answers, O.brute(od, oq_of(P.L1, queries), O.KNN, ks=np.full(16, k)))
        for _, d in answers:
            assert d.tolist() == sorted(d.tolist())


@pytest.mark.parametrize("metric", [P.L2, P.EDIT])
def test_batch_equals_sequential(metric):
    rng = np.random.default_rng(32)
    tree, _, payloads, _ = make_index(150, metric=metric, nc=3, seed=4)
    eng = P.BatchSearcher(tree)
    queries = [payloads[int(i)] for i in rng.integers(0, 150, 20)]
    radii = rng.uniform(0.05, 0.4, 20) if metric != P.EDIT else rng.integers(0, 6, 20).astype(float)
    batch, _ = eng.range_batch(queries, radii)
    for q in range(20):
        single, _ = eng.range_batch([queries[q]], [radii[q]])
        assert pairs(single)[0] == pairs(batch)[q]
    ks = rng.integers(1, 9, 20)
    batch, _ = eng.knn_batch(queries, ks)
    for q in range(20):
        single, _ = eng.knn_batch([queries[q]], [int(ks[q])])
        assert pairs(single)[0] == pairs(batch)[q]


def test_runtime_never_changes_answers():
    rng = np.random.default_rng(33)
    tree, _, payloads, _ = make_index(200, nc=4, seed=5)
    queries = [payloads[int(i)] for i in rng.integers(0, 200, 24)]
    results = []
    for workers in (1, 4, 8):
        eng = P.BatchSearcher(tree, runtime=P.ParallelRuntime(workers=workers))
        results.append((pairs(eng.range_batch(queries, 0.25)[0]), pairs(eng.knn_batch(queries, 5)[0])))
    assert results[0] == results[1] == results[2]


def test_tight_budget_still_exact_and_logged():
    rng = np.random.default_rng(34)
    tree, _, payloads, _ = make_index(300, nc=4, seed=6)
    queries = [payloads[int(i)] for i in rng.integers(0, 300, 32)]
    radii = rng.uniform(0.05, 0.5, 32)
    wide, _ = P.BatchSearcher(tree).range_batch(queries, radii)
    tight_eng = P.BatchSearcher(tree, memory_units=16)
    tight, stats = tight_eng.range_batch(queries, radii)
    assert pairs(wide) == pairs(tight)
    assert stats.peak_units <= 16
    widek, _ = P.BatchSearcher(tree).knn_batch(queries, 7)
    tightk, kstats = tight_eng.knn_batch(queries, 7)
    assert pairs(widek) == pairs(tightk)
    assert kstats.peak_units <= 16
    tree2, _, payloads2, _ = make_index(400, nc=4, seed=7)
    _, s2 = P.BatchSearcher(tree2, memory_units=64).range_batch(payloads2[:8], 0.2)
    assert s2.size_limits
    for layer, limit in s2.size_limits.items():
        assert limit == P.level_size_limit(64, tree2.nc, tree2.split_rounds, layer)


def test_pruning_disabled_same_answers_more_work():
    rng = np.random.default_rng(35)
    tree, _, payloads, _ = make_index(160, nc=4, seed=8)
    queries = [payloads[int(i)] for i in rng.integers(0, 160, 10)]
    on, off = P.BatchSearcher(tree, pruning=True), P.BatchSearcher(tree, pruning=False)
    a_on, s_on = on.range_batch(queries, 0.15)
    a_off, s_off = off.range_batch(queries, 0.15)
    assert pairs(a_on) == pairs(a_off)
    assert np.all(s_off.verified == tree.n)
    assert s_on.total_verified < s_off.total_verified
    assert pairs(on.knn_batch(queries, 4)[0]) == pairs(off.knn_batch(queries, 4)[0])


def test_tombstoned_entries_never_returned():
    rng = np.random.default_rng(36)
    tree, _, payloads, od = make_index(120, nc=3, seed=9)
    dead = {int(i) for i in rng.choice(120, 30, replace=False)}
    for obj in dead:
        tree.tombstone[tree.entry_pos_of_id(obj)] = 1
    eng = P.BatchSearcher(tree)
    queries = [payloads[int(i)] for i in rng.integers(0, 120, 15)]
    dead_rows = np.zeros(120, np.uint8)
    dead_rows[list(dead)] = 1
    oq = oq_of(P.L2, queries)
    answers, _ = eng.range_batch(queries, 0.4)
    assert_matches(answers, O.brute(od, oq, O.RANGE, radii=np.full(15, 0.4), dead_rows=dead_rows))
    answers, _ = eng.knn_batch(queries, 6)
    assert_matches(answers, O.brute(od, oq, O.KNN, ks=np.full(15, 6), dead_rows=dead_rows))
    for ids, _ in answers:
        assert not (set(ids.tolist()) & dead)


@pytest.mark.parametrize("probe", ["node_major", "per_query"])
@pytest.mark.parametrize("metric,dim,n,nc", [(P.L2, 64, 20000, 4), (P.L1, 32, 6000, 6)])
def test_knn_probe_paths_exact_with_tombstones(probe, metric, dim, n, nc, monkeypatch):
    """kNN radius probe: node-major (k_probe_path/dist/select, D >= 16) and
    per-query (k_probe) both give exact answers, with tombstoned entries in
    the probed nodes and k from 1 to beyond a node's size."""
    if probe == "per_query":
        monkeypatch.setenv("GTS_PROBE_PERQUERY", "1")
    else:
        monkeypatch.delenv("GTS_PROBE_PERQUERY", raising=False)
    rng = np.random.default_rng(37)
    # (20000, 4): the probe node sits two levels down (5000 -> 1250 entries)
    # and takes its sibling ring; (6000, 6): level-1 nodes hold < 1024, so
    # the root itself is probed
    mat = P.generate_clustered(n, dim, 12, seed=38, spread=0.05)
    ds = P.Dataset.from_vectors(mat, metric)
    tree = P.build(ds, P.TreeConfig(node_capacity=nc, seed=2))
    dead = rng.choice(n, n // 7, replace=False)
    for obj in dead:
        tree.tombstone[tree.entry_pos_of_id(int(obj))] = 1
    dead_rows = np.zeros(n, np.uint8)
    dead_rows[dead] = 1
    qi = rng.integers(0, n, 40)
    queries = [mat[i] + rng.normal(0, 0.01, dim) for i in qi]
    od = O.Payloads({P.L1: 1, P.L2: 2}[metric], vec=mat)
    oq = O.Payloads({P.L1: 1, P.L2: 2}[metric], vec=np.array(queries))
    eng = P.BatchSearcher(tree)
    for k in (1, 10, 100, 1500):
        got, _ = eng.knn_batch(queries, k)
        assert_matches(got, O.brute(od, oq, O.KNN, ks=np.full(40, k), dead_rows=dead_rows))


@pytest.mark.parametrize("metric", [P.EDIT, P.L2])
def test_knn_verified_stats_semantics(metric):
    """kNN `verified` counts are the device pass's own: the
    live entries that pass lemma 1 under the query's radius as it shrinks
    during the pass, not the reference's count under its witness-pool bound
    (search.py:540-570), which depends on the reference's visiting order.
    What holds for both: every answer was verified, the count never exceeds
    the live collection, and pruning off verifies every live entry."""
    tree, ds, payloads, od = make_index(600, metric=metric, nc=5, seed=4)
    q = [payloads[i] for i in range(0, 600, 37)]
    eng = P.BatchSearcher(tree)
    ans, st = eng.knn_batch(q, 7)
    assert np.all(st.verified >= np.array([a[0].size for a in ans]))
    assert np.all(st.verified <= 600)
    _, st_off = P.BatchSearcher(tree, pruning=False).knn_batch(q, 7)
    assert np.all(st_off.verified == 600)
    # and the range stats stay the reference's (edit: equal; floats: >=)
    ref = O.search(O.build(od, 5, 4), od, oq_of(metric, q), O.RANGE, radii=np.full(len(q), 3.0 if metric == P.EDIT else 0.2))
    _, sr = eng.range_batch(q, 3.0 if metric == P.EDIT else 0.2)
    if metric == P.EDIT:
        assert np.array_equal(sr.verified, ref.verified)
    else:
        assert np.all(sr.verified >= ref.verified)
