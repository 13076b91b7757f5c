"""Host-side logic of the product: native builder vs the reference's trees,
scheduling helpers, and the C ABI surface (no GPU needed)."""

import os
import re

import numpy as np
import pytest

import paper_2404_00966_b200 as P
from paper_2404_00966_b200 import _lib
from conftest import ROOT, TREES, decode_strings, load_golden

TREE_FIELDS = ["pivot_id", "pivot_row", "min_dis", "max_dis", "pos", "size", "rows", "dis"]


def dataset_of(g):
    met = int(g["metric"])
    if met == 0:
        return P.Dataset.from_strings(decode_strings(g["data_codes"], g["data_off"]), P.EDIT, ids=g["ids"])
    return P.Dataset.from_vectors(g["data_vec"], {1: P.L1, 2: P.L2}[met], ids=g["ids"])


@pytest.mark.parametrize("name", TREES)
def test_native_builder_matches_reference_tree(name):
    g = load_golden(name)
    t = P.build(dataset_of(g), P.TreeConfig(int(g["nc"]), int(g["seed"])))
    assert t.levels == int(g["levels"]) and t.split_rounds == int(g["split_rounds"])
    for f in TREE_FIELDS:
        assert np.array_equal(getattr(t, f), g[f]), f


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "gts.h")).read()
    declared = set(re.findall(r"\b(gts_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(_lib.EXPORTED)
    L = _lib.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert L.gts_version().decode().startswith("gts-b200")


def test_tree_height_known_values():
    assert P.tree_height(10, 2) == (3, 2)
    assert P.tree_height(611756, 20) == (4, 3)
    assert P.tree_height(1, 2) == (0, 0)
    assert P.tree_height(20 ** 4 - 1, 20) == (3, 2)
    assert P.tree_height(20 ** 4, 20) == (4, 3)
    mh, sp = np.zeros(1, np.int64), np.zeros(1, np.int64)
    for n, nc in [(10, 2), (611756, 20), (1, 2), (12_500_000, 20), (100_000_000, 20)]:
        _lib.check(_lib.lib().gts_tree_height(n, nc, _lib.ptr(mh, _lib._i64p), _lib.ptr(sp, _lib._i64p)))
        assert (int(mh[0]), int(sp[0])) == P.tree_height(n, nc)


def test_level_size_limit_formula():
    assert P.level_size_limit(8000, 20, 4, 1) == 100
    assert P.level_size_limit(1000, 20, 2, 1) == 25
    assert P.level_size_limit(1000, 20, 2, 2) == 50
    assert P.level_size_limit(1, 20, 2, 1) == 1
    with pytest.raises(ValueError):
        P.level_size_limit(1000, 20, 2, 0)


def test_query_groups_first_fit():
    assert P.compute_query_groups([2, 99, 3], 10) == [[0, 2], [1]]
    assert P.compute_query_groups([5, 5, 5], 10) == [[0, 1], [2]]


def test_predicates_boundaries():
    assert not P.object_prunable(entry_dis=5.0, dqp=3.0, radius=2.0)
    assert P.object_prunable(entry_dis=5.0, dqp=3.0, radius=1.9)
    assert not P.node_prunable_range(dqp=5.0, radius=1.0, min_dis=6.0, max_dis=9.0)
    assert P.node_prunable_knn(dqp=5.0, bound=1.0, min_dis=6.0, max_dis=9.0)
    assert P.current_kth_bound(np.array([1.0, 2.0, 7.0]), 4) == float("inf")


def test_capacity_below_fanout_rejected():
    ds = P.Dataset.from_vectors(np.random.default_rng(0).uniform(size=(50, 2)), P.L2)
    t = P.build(ds, P.TreeConfig(node_capacity=8))
    with pytest.raises(P.BudgetError):
        P.BatchSearcher(t, memory_units=7)
    P.BatchSearcher(t, memory_units=8)


def test_query_validation_raises_reference_types():
    ds = P.Dataset.from_vectors(np.random.default_rng(0).uniform(size=(30, 2)), P.L2)
    t = P.build(ds, P.TreeConfig(node_capacity=4))
    eng = P.BatchSearcher(t)
    q = [ds.mat[0], ds.mat[1]]
    with pytest.raises(ValueError):
        eng.range_batch(q, [-0.5, 0.1])
    with pytest.raises(ValueError):
        eng.knn_batch(q, 0)
    with pytest.raises(ValueError):
        eng.range_batch(q + [ds.mat[2]], [0.1, 0.2])
    with pytest.raises(P.MetricMismatchError):
        eng.range_batch([np.zeros(3)], 0.1)


def test_empty_index_answers_empty():
    ds = P.Dataset.from_vectors(np.empty((0, 2)), P.L2)
    t = P.build(ds, P.TreeConfig(node_capacity=4))
    ans, stats = P.BatchSearcher(t).range_batch([np.array([0.5, 0.5])], 10.0)
    assert ans[0][0].size == 0
    ans, _ = P.BatchSearcher(t).knn_batch([np.array([0.5, 0.5])], 3)
    assert ans[0][0].size == 0
