"""In-place inserts into leaf slack (gts_index_insert, csrc/updates.cuh;
SURVEY.md §8(f2)) under the reference's StreamingIndex rules
(updates.py:109-158): after every batch of deletes / inserts / re-inserts /
deletes of pending objects, range and kNN answers must equal the oracle's
brute force over the tracked live set (oracle.py:19-36), with the tree
pruning the placed objects (placed_count > 0) and objects that do not fit
falling back to the device cache."""

import ctypes as C

import numpy as np
import pytest

import paper_2404_00966_b200 as P
from oracle import oracle as O
from paper_2404_00966_b200 import _lib

pytestmark = pytest.mark.gpu


def live_brute(metric, live, queries, radii, ks):
    ids = np.array(sorted(live), dtype=np.int64)
    if metric == P.EDIT:
        od = O.Payloads.from_strings([live[i] for i in ids], ids=ids)
        oq = O.Payloads.from_strings(queries)
    else:
        code = {P.L1: O.L1, P.L2: O.L2}[metric]
        od = O.Payloads(code, vec=np.array([live[i] for i in ids]), ids=ids)
        oq = O.Payloads(code, vec=np.array(queries))
    return (O.brute(od, oq, O.RANGE, radii=radii, threads=8).answers(),
            O.brute(od, oq, O.KNN, ks=ks, threads=8).answers())


def check(si, metric, live, queries, radii, ks, pruning=True):
    wr, wk = live_brute(metric, live, queries, radii, ks)
    gr, _ = si.query_range(queries, radii, pruning=pruning)
    gk, _ = si.query_knn(queries, ks, pruning=pruning)
    for g, w in zip(gr + gk, wr + wk):
        assert np.array_equal(g[0], w[0]) and np.array_equal(g[1], w[1])


def make(kind, n, rng):
    if kind == "words":
        strs = P.generate_sequences(n, seed=1, min_len=1, max_len=20, alphabet="abcdefghijklmnop")
        return P.EDIT, strs, lambda: "".join(rng.choice(list("abcdefghijklmnop"), int(rng.integers(1, 18))))
    if kind == "dna":
        strs = P.generate_sequences(n, seed=2, min_len=60, max_len=60, alphabet="ACGT")
        return P.EDIT, strs, lambda: "".join(rng.choice(list("ACGT"), 60))
    D = {"l2_128": 128, "l1_32": 32, "l2_2": 2}[kind]
    metric = P.L1 if kind == "l1_32" else P.L2
    centers = rng.uniform(0, 1, (40, D)).astype(np.float32)
    mat = (centers[rng.integers(0, 40, n)] + rng.normal(0, 0.05, (n, D))).astype(np.float32).astype(np.float64)
    new = lambda: (centers[rng.integers(0, 40)] + rng.normal(0, 0.05, D)).astype(np.float32).astype(np.float64)
    return metric, list(mat), new


@pytest.mark.parametrize("kind", ["words", "dna", "l2_128", "l1_32", "l2_2"])
def test_in_place_inserts_stay_exact(kind):
    rng = np.random.default_rng(3)
    n = 12000
    metric, payloads, new = make(kind, n, rng)
    ds = (P.Dataset.from_strings(payloads, metric) if metric == P.EDIT else
          P.Dataset.from_vectors(np.array(payloads), metric))
    si = P.StreamingIndex(ds, P.TreeConfig(20, 0), cache_capacity=5000)
    live = {i: payloads[i] for i in range(n)}
    next_id = n
    nq = 24
    for rnd in range(4):
        dels = [int(i) for i in rng.choice(sorted(live), 150, replace=False)]
        ins = []
        for oid in dels[:60]:              # re-insert deleted ids with new payloads
            ins.append((oid, new()))
        for _ in range(300):               # fresh ids
            ins.append((next_id, new()))
            next_id += 1
        si.batch_update(inserts=ins, deletes=dels)
        for oid in dels:
            live.pop(oid)
        for oid, p in ins:
            live[oid] = p
        # delete some pending (placed) objects again
        pend = [i for i, _ in ins[60:]]
        for oid in rng.choice(pend, 40, replace=False):
            si.delete(int(oid))
            live.pop(int(oid))
        assert si.rebuild_count == 0
        assert si.placed_count > 0.5 * len(si.pending)
        qi = rng.choice(sorted(live), nq, replace=False)
        queries = [live[int(i)] for i in qi[: nq // 2]] + [new() for _ in range(nq - nq // 2)]
        if metric == P.EDIT:
            radii = rng.integers(0, 4, nq).astype(float)
        else:
            radii = rng.uniform(0.05, 0.4 if kind != "l2_128" else 0.8, nq)
        ks = rng.integers(1, 30, nq)
        check(si, metric, live, queries, radii, ks)
        if rnd == 3:
            check(si, metric, live, queries, radii, ks, pruning=False)


def test_full_leaves_fall_back_to_the_cache():
    """Many inserts into one region: the leaves fill up, the rest stays in the
    device cache, answers stay exact."""
    rng = np.random.default_rng(4)
    mat = rng.uniform(0, 1, (3000, 4)).astype(np.float32).astype(np.float64)
    si = P.StreamingIndex(P.Dataset.from_vectors(mat, P.L2), P.TreeConfig(20, 0), cache_capacity=4000)
    live = {i: mat[i] for i in range(3000)}
    spot = np.array([0.5, 0.5, 0.5, 0.5])
    ins = [(3000 + j, (spot + rng.normal(0, 0.01, 4)).astype(np.float32).astype(np.float64)) for j in range(1500)]
    si.batch_update(inserts=ins)
    live.update(dict(ins))
    assert 0 < si.placed_count < len(ins)
    q = [spot, spot + 0.02, mat[5]]
    check(si, P.L2, live, q, np.array([0.02, 0.05, 0.1]), np.array([10, 200, 1]))


def test_insert_abi_reports_unplaceable_items():
    strs = P.generate_sequences(2000, seed=5, min_len=3, max_len=10, alphabet="abc")
    tree = P.build(P.Dataset.from_strings(strs, P.EDIT), P.TreeConfig(20, 0))
    h = tree.device_index(0).h
    items = P.Dataset.from_strings(["ab", "zzz", "a" * 40, "abcabc"], P.EDIT, ids=np.array([5000, 5001, 5002, 5003]))
    from paper_2404_00966_b200.tree import _c_dataset
    c_ds, keep = _c_dataset(items)
    slots = np.zeros(4, dtype=np.int32)
    _lib.check(_lib.lib().gts_index_insert(h, C.byref(c_ds), _lib.ptr(slots, _lib._i32p), None))
    assert slots[0] >= 0 and slots[3] >= 0      # placed
    assert slots[1] == -1 and slots[2] == -1    # symbol outside the alphabet; longer than a slot
    bad = np.array([0], dtype=np.int32)          # a slot of the reference tree, not an insert
    assert _lib.lib().gts_index_erase(h, _lib.ptr(bad, _lib._i32p), 1, None) == _lib.GTS_EINVAL
