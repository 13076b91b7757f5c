"""Device path vs the reference: golden fixtures from the reference itself
and the C oracle (oracle/) on larger seeded inputs.  Runs through the
C ABI (libgts.so) via the drop-in BatchSearcher.

Parity bar (BASELINE.json north_star): range id sets identical; distances
bit-identical (float64 in numpy's order / exact integers); kNN = canonical
brute-force (distance, id) top-k, distance lists identical to the
reference engine's.
"""

import numpy as np
import pytest

import paper_2404_00966_b200 as P
from conftest import TIGHT_UNITS, TREES, decode_strings, load_golden
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["default", "rowwise", "grouped_alt", "smem_text"], autouse=True)
def leaf_path(request, monkeypatch):
    """Every test runs on each leaf-verification path: default (k_leaf_edit;
    k_leafgroup_mma2 / k_leafgroup_tile for vectors), row-wise vectors
    (k_verify, GTS_NO_GROUPED=1), the grouped alternates (k_leafgroup_edit,
    warp-per-row k_leafgroup_vec) and the smem-text DP of k_leaf_edit."""
    for k in ("GTS_NO_GROUPED", "GTS_EDIT_GROUPED", "GTS_EDIT_SMEM_TEXT", "GTS_VEC_ROWWARP"):
        monkeypatch.delenv(k, raising=False)
    if request.param == "rowwise":
        monkeypatch.setenv("GTS_NO_GROUPED", "1")
    elif request.param == "grouped_alt":
        monkeypatch.setenv("GTS_EDIT_GROUPED", "1")
        monkeypatch.setenv("GTS_VEC_ROWWARP", "1")
    elif request.param == "smem_text":
        monkeypatch.setenv("GTS_EDIT_SMEM_TEXT", "1")
    return request.param


def setup(name):
    g = load_golden(name)
    met = int(g["metric"])
    if met == 0:
        ds = P.Dataset.from_strings(decode_strings(g["data_codes"], g["data_off"]), P.EDIT, ids=g["ids"])
        queries = decode_strings(g["query_codes"], g["query_off"])
        od = O.Payloads(0, codes=g["data_codes"], off=g["data_off"], ids=g["ids"])
        oq = O.Payloads(0, codes=g["query_codes"], off=g["query_off"])
    else:
        metric = {1: P.L1, 2: P.L2}[met]
        ds = P.Dataset.from_vectors(g["data_vec"], metric, ids=g["ids"])
        queries = [g["query_vec"][i] for i in range(g["query_vec"].shape[0])]
        od = O.Payloads(met, vec=g["data_vec"], ids=g["ids"])
        oq = O.Payloads(met, vec=g["query_vec"])
    tree = P.build(ds, P.TreeConfig(int(g["nc"]), int(g["seed"])))
    return g, ds, tree, queries, od, oq


def csr(answers):
    return (np.array([a[0].size for a in answers]),
            np.concatenate([a[0] for a in answers]) if answers else np.empty(0, np.int64),
            np.concatenate([a[1] for a in answers]) if answers else np.empty(0))


@pytest.mark.parametrize("name", TREES)
def test_range_matches_reference(name):
    g, ds, tree, queries, _, _ = setup(name)
    ans, st = P.BatchSearcher(tree).range_batch(queries, g["radii"])
    c, i, d = csr(ans)
    assert np.array_equal(c, g["range_wide_counts"])
    assert np.array_equal(i, g["range_wide_ids"])
    assert np.array_equal(d, g["range_wide_dis"])          # bit-exact float64
    # same tree + same predicates -> same work counters (fp32 slack can only add)
    assert np.all(st.verified >= g["range_wide_verified"])
    assert np.all(st.pruned_nodes <= g["range_wide_pruned"])
    if int(g["metric"]) == 0:
        assert np.array_equal(st.verified, g["range_wide_verified"])
        assert np.array_equal(st.pruned_nodes, g["range_wide_pruned"])


@pytest.mark.parametrize("name", TREES)
def test_range_tight_budget(name):
    g, ds, tree, queries, _, _ = setup(name)
    units = TIGHT_UNITS[name]
    ans, st = P.BatchSearcher(tree, memory_units=units).range_batch(queries, g["radii"])
    c, i, d = csr(ans)
    assert np.array_equal(i, g["range_tight_ids"]) and np.array_equal(d, g["range_tight_dis"])
    assert st.peak_units <= units
    assert st.size_limits == {int(a): int(b) for a, b in g["range_tight_limits"]}


@pytest.mark.parametrize("name", TREES)
def test_knn_canonical_and_reference_distances(name):
    g, ds, tree, queries, od, oq = setup(name)
    ans, _ = P.BatchSearcher(tree).knn_batch(queries, g["ks"])
    c, i, d = csr(ans)
    want = O.brute(od, oq, O.KNN, ks=g["ks"])
    assert np.array_equal(c, want.counts)
    assert np.array_equal(i, want.ids)       # canonical (distance, id) order
    assert np.array_equal(d, want.dis)
    assert np.array_equal(d, g["knn_wide_dis"])  # = the reference engine's distances


@pytest.mark.parametrize("name", TREES)
def test_tombstones_and_pruning_off(name):
    g, ds, tree, queries, od, oq = setup(name)
    tree.tombstone[:] = g["tombstone"]
    eng = P.BatchSearcher(tree)
    ans, st = eng.range_batch(queries, g["radii"])
    c, i, d = csr(ans)
    assert np.array_equal(i, g["dead_range_wide_ids"]) and np.array_equal(d, g["dead_range_wide_dis"])
    dead = np.zeros(ds.n, np.uint8)
    dead[tree.rows[tree.tombstone == 1]] = 1
    want = O.brute(od, oq, O.KNN, ks=g["ks"], dead_rows=dead)
    ans, _ = eng.knn_batch(queries, g["ks"])
    c, i, d = csr(ans)
    assert np.array_equal(i, want.ids) and np.array_equal(d, want.dis)
    off = P.BatchSearcher(tree, pruning=False)
    ans, st = off.range_batch(queries, g["radii"])
    c, i, d = csr(ans)
    assert np.array_equal(i, g["dead_nopr_range_ids"])
    assert np.array_equal(st.verified, g["dead_nopr_range_verified"])
    ans, _ = off.knn_batch(queries, g["ks"])
    c, i, d = csr(ans)
    assert np.array_equal(i, want.ids) and np.array_equal(d, want.dis)


def test_pair_distances_match_reference(golden_metrics):
    m = golden_metrics
    ao, bo, ac, bc = m["edit_a_off"], m["edit_b_off"], m["edit_a_codes"], m["edit_b_codes"]
    a = decode_strings(ac, ao)
    b = decode_strings(bc, bo)
    assert np.array_equal(P.pair_distances(P.EDIT, a, b), m["edit_d"])
    for k in m.files:
        if k.startswith("vec") and k.endswith("_l1"):
            base = k[:-3]
            for met, key in ((P.L1, "_l1"), (P.L2, "_l2")):
                got = P.pair_distances(met, m[base + "_a"], m[base + "_b"])
                assert np.array_equal(got, m[base + key]), base + key


# -- larger seeded workloads against the C oracle --------------------------

def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def string_queries(strings, nq, rng, alphabet):
    out = [strings[int(i)] for i in rng.integers(0, len(strings), nq // 2)]
    for i in rng.integers(0, len(strings), nq - nq // 2):
        s = list(strings[int(i)])
        for _ in range(int(rng.integers(1, 3))):
            c = alphabet[int(rng.integers(0, len(alphabet)))]
            if s and rng.integers(0, 2):
                s[int(rng.integers(0, len(s)))] = c
            else:
                s.insert(int(rng.integers(0, len(s) + 1)), c)
        out.append("".join(s))
    return out


def check_against_oracle(ds, tree, queries, od, oq, radii, ks, threads=8):
    eng = P.BatchSearcher(tree)
    ans, st = eng.range_batch(queries, radii)
    c, i, d = csr(ans)
    want = O.brute(od, oq, O.RANGE, radii=radii, threads=threads)
    assert np.array_equal(c, want.counts)
    assert np.array_equal(i, want.ids)
    assert np.array_equal(d, want.dis)
    ans, _ = eng.knn_batch(queries, ks)
    c, i, d = csr(ans)
    want = O.brute(od, oq, O.KNN, ks=ks, threads=threads)
    assert np.array_equal(c, want.counts)
    assert np.array_equal(i, want.ids)
    assert np.array_equal(d, want.dis)


def test_tloc_like_l2_100k():
    rng = np.random.default_rng(3)
    mat = f32(P.generate_uniform(100_000, 2, seed=12))
    ds = P.Dataset.from_vectors(mat, P.L2)
    tree = P.build(ds, P.TreeConfig(20, 0))
    q = f32(P.generate_uniform(300, 2, seed=13))
    radii = np.full(300, 0.0582588)
    check_against_oracle(ds, tree, list(q), O.Payloads(O.L2, vec=mat), O.Payloads(O.L2, vec=q), radii,
                         rng.integers(1, 40, 300))


def test_l1_32d_clustered():
    rng = np.random.default_rng(4)
    mat = f32(P.generate_clustered(30_000, 32, 50, seed=5, spread=0.05))
    ds = P.Dataset.from_vectors(mat, P.L1)
    tree = P.build(ds, P.TreeConfig(20, 1))
    q = np.concatenate([mat[rng.integers(0, 30_000, 40)], f32(rng.uniform(0, 1, (40, 32)))])
    check_against_oracle(ds, tree, list(q), O.Payloads(O.L1, vec=mat), O.Payloads(O.L1, vec=q),
                         rng.uniform(0.5, 3.0, 80), rng.integers(1, 101, 80))


def test_l2_128d_not_fp32_exact():
    # raw float64 payloads: the device keeps a float64 copy for the exact recheck
    rng = np.random.default_rng(5)
    mat = P.generate_clustered(5_000, 128, 20, seed=6, spread=0.05)
    ds = P.Dataset.from_vectors(mat, P.L2)
    tree = P.build(ds, P.TreeConfig(10, 2))
    q = np.concatenate([mat[rng.integers(0, 5_000, 20)], rng.uniform(0, 1, (20, 128))])
    check_against_oracle(ds, tree, list(q), O.Payloads(O.L2, vec=mat), O.Payloads(O.L2, vec=q),
                         rng.uniform(0.2, 1.5, 40), rng.integers(1, 20, 40))


def test_words_like_edit():
    rng = np.random.default_rng(6)
    alpha = "abcdefghijklmnopqrstuvwxyz"
    strs = P.generate_sequences(40_000, seed=21, min_len=1, max_len=34, alphabet=alpha)
    ds = P.Dataset.from_strings(strs, P.EDIT)
    tree = P.build(ds, P.TreeConfig(20, 3))
    q = string_queries(strs, 120, rng, alpha)
    check_against_oracle(ds, tree, q, O.Payloads.from_strings(strs), O.Payloads.from_strings(q),
                         rng.integers(0, 4, 120).astype(float), rng.integers(1, 16, 120))


def test_dna_108_edit():
    rng = np.random.default_rng(7)
    strs = P.generate_sequences(8_000, seed=22, min_len=108, max_len=108, alphabet="ACGT")
    ds = P.Dataset.from_strings(strs, P.EDIT)
    tree = P.build(ds, P.TreeConfig(20, 4))
    q = string_queries(strs, 24, rng, "ACGT")
    check_against_oracle(ds, tree, q, O.Payloads.from_strings(strs), O.Payloads.from_strings(q),
                         rng.integers(0, 60, 24).astype(float), rng.integers(1, 12, 24))


def test_edge_cases_strings():
    # empty strings, long strings (generic multi-word path), symbols absent
    # from the index alphabet, duplicates, radius 0, k > n
    rng = np.random.default_rng(8)
    strs = ["", "a", "ab", "ab", "ba", "abc" * 60, "abd" * 60, "x" * 300, "é漢", "漢é"] + \
        P.generate_sequences(300, seed=9, min_len=0, max_len=200, alphabet="abcé漢")
    ds = P.Dataset.from_strings(strs, P.EDIT)
    tree = P.build(ds, P.TreeConfig(3, 5))
    q = ["", "ab", "zzz", "abc" * 61, "é", "q" * 400] + string_queries(strs, 20, rng, "abcé漢z")
    nq = len(q)
    check_against_oracle(ds, tree, q, O.Payloads.from_strings(strs), O.Payloads.from_strings(q),
                         np.concatenate([[0.0, 0.0, 3.0, 5.0, 1.0, 50.0], rng.integers(0, 40, nq - 6)]).astype(float),
                         np.concatenate([[1, 2, 400, 5, 3, 1], rng.integers(1, 30, nq - 6)]))


def test_edge_cases_strings_mixed_widths():
    # queries of 0..128 symbols (1-4 pattern words mixed inside one warp's
    # row group), empty and duplicate objects, overfull leaves, tombstones
    rng = np.random.default_rng(18)
    alpha = "abcdefghij"
    strs = ["", "", "a", "abc" * 40] + P.generate_sequences(3000, seed=19, min_len=0, max_len=140, alphabet=alpha)
    ds = P.Dataset.from_strings(strs, P.EDIT)
    tree = P.build(ds, P.TreeConfig(6, 7))
    q = ["", "a", "abc" * 40 + "ab", "j" * 33, "ab" * 32] + \
        P.generate_sequences(40, seed=20, min_len=0, max_len=128, alphabet=alpha + "z")
    nq = len(q)
    check_against_oracle(ds, tree, q, O.Payloads.from_strings(strs), O.Payloads.from_strings(q),
                         rng.integers(0, 70, nq).astype(float), rng.integers(1, 40, nq))


def test_edge_cases_vectors():
    mat = np.array([[0.0, 0.0], [1.0, 1.0], [0.0, 0.0], [2.0, 2.0]])
    ds = P.Dataset.from_vectors(mat, P.L2)
    tree = P.build(ds, P.TreeConfig(node_capacity=2, seed=0))
    ans, _ = P.BatchSearcher(tree).range_batch([np.array([0.0, 0.0])], 0.0)
    assert ans[0][0].tolist() == [0, 2] and ans[0][1].tolist() == [0.0, 0.0]
    ans, _ = P.BatchSearcher(tree).knn_batch([np.array([0.0, 0.0])], 25)
    assert ans[0][0].tolist() == [0, 2, 1, 3]
    one = P.Dataset.from_vectors(np.array([[0.5, 0.5]]), P.L2)
    t1 = P.build(one, P.TreeConfig(4))
    assert t1.levels == 1
    ans, _ = P.BatchSearcher(t1).knn_batch([np.array([0.0, 0.0])], 3)
    assert ans[0][0].tolist() == [0]


def test_streaming_index_matches_live_set():
    rng = np.random.default_rng(10)
    alpha = "ACGT"
    strs = P.generate_sequences(3000, seed=11, min_len=20, max_len=40, alphabet=alpha)
    ds = P.Dataset.from_strings(strs, P.EDIT)
    si = P.StreamingIndex(ds, P.TreeConfig(8, 0), cache_capacity=64)
    live = dict(enumerate(strs))
    next_id = 3000
    for step in range(6):
        for oid in rng.choice(sorted(live), 40, replace=False):
            si.delete(int(oid))
            del live[int(oid)]
        for _ in range(30):
            s = "".join(alpha[i] for i in rng.integers(0, 4, int(rng.integers(20, 41))))
            si.insert(next_id, s)
            live[next_id] = s
            next_id += 1
        q = string_queries(list(live.values()), 10, rng, alpha)
        ids = np.array(sorted(live), dtype=np.int64)
        od = O.Payloads.from_strings([live[i] for i in ids], ids=ids)
        oq = O.Payloads.from_strings(q)
        got, _ = si.query_range(q, 8.0)
        want = O.brute(od, oq, O.RANGE, radii=np.full(10, 8.0))
        c, i, d = csr(got)
        assert np.array_equal(i, want.ids) and np.array_equal(d, want.dis)
        got, _ = si.query_knn(q, 7)
        want = O.brute(od, oq, O.KNN, ks=np.full(10, 7))
        c, i, d = csr(got)
        assert np.array_equal(i, want.ids) and np.array_equal(d, want.dis)
    assert si.rebuild_count >= 1


# -- tensor-core (tcgen05 tf32) L2 verification path ------------------------

@pytest.mark.parametrize("dim,clustered", [(64, True), (100, False), (128, True), (128, False)])
def test_l2_tensor_core_path_exact(dim, clustered):
    """L2 with D >= 32 verifies leaf blocks with a tf32 tcgen05 MMA plus an
    exact float64 recheck; answers must equal brute force bit-exactly."""
    rng = np.random.default_rng(dim + 7 * clustered)
    n = 30_000
    if clustered:
        mat = f32(P.generate_clustered(n, dim, 60, seed=dim, spread=0.05))
        q = mat[rng.integers(0, n, 200)] + f32(rng.normal(0, 0.01, (200, dim)))
    else:
        mat = f32(P.generate_uniform(n, dim, seed=dim))
        q = f32(rng.uniform(0, 1, (200, dim)))
    q = f32(q)
    ds = P.Dataset.from_vectors(mat, P.L2)
    tree = P.build(ds, P.TreeConfig(20, 1))
    radii = rng.uniform(0.2, 0.9, 200) * (1.0 if clustered else np.sqrt(dim / 6.0))
    check_against_oracle(ds, tree, list(q), O.Payloads(O.L2, vec=mat), O.Payloads(O.L2, vec=q), radii,
                         rng.integers(1, 30, 200))


def test_streaming_index_vectors_and_new_symbols():
    """Device pending-insert cache: L2 vectors, and strings whose inserts bring
    symbols the index alphabet lacks (the pair-distance fallback)."""
    rng = np.random.default_rng(12)
    mat = f32(P.generate_uniform(2000, 8, seed=3))
    si = P.StreamingIndex(P.Dataset.from_vectors(mat, P.L2), P.TreeConfig(6, 0), cache_capacity=200)
    live = {i: mat[i] for i in range(2000)}
    nid = 5000
    for step in range(4):
        for oid in rng.choice(sorted(live), 25, replace=False):
            si.delete(int(oid))
            del live[int(oid)]
        for _ in range(40):
            v = f32(rng.uniform(0, 1, 8))
            si.insert(nid, v)
            live[nid] = v
            nid += 1
        # re-insert a deleted id with a new payload (the tombstone hides the stale entry)
        q = f32(rng.uniform(0, 1, (12, 8)))
        ids = np.array(sorted(live), dtype=np.int64)
        od = O.Payloads(O.L2, vec=np.array([live[i] for i in ids]), ids=ids)
        oq = O.Payloads(O.L2, vec=q)
        got, _ = si.query_range(list(q), 0.3)
        want = O.brute(od, oq, O.RANGE, radii=np.full(12, 0.3))
        c, i, d = csr(got)
        assert np.array_equal(i, want.ids) and np.array_equal(d, want.dis)
        got, _ = si.query_knn(list(q), 9)
        want = O.brute(od, oq, O.KNN, ks=np.full(12, 9))
        c, i, d = csr(got)
        assert np.array_equal(i, want.ids) and np.array_equal(d, want.dis)
    # strings: a pending insert with a symbol outside the alphabet
    strs = P.generate_sequences(500, seed=4, min_len=5, max_len=15, alphabet="ACGT")
    si = P.StreamingIndex(P.Dataset.from_strings(strs, P.EDIT), P.TreeConfig(5, 0), cache_capacity=50)
    si.insert(900, "ACGTZZ")
    si.insert(901, "ACGTAC")
    si.delete(3)
    live = {i: s for i, s in enumerate(strs) if i != 3}
    live.update({900: "ACGTZZ", 901: "ACGTAC"})
    ids = np.array(sorted(live), dtype=np.int64)
    q = ["ACGTZZ", "ACG", "TTTTT", "Z"]
    od = O.Payloads.from_strings([live[i] for i in ids], ids=ids)
    oq = O.Payloads.from_strings(q)
    got, _ = si.query_knn(q, 5)
    want = O.brute(od, oq, O.KNN, ks=np.full(4, 5))
    c, i, d = csr(got)
    assert np.array_equal(i, want.ids) and np.array_equal(d, want.dis)
    got, _ = si.query_range(q, 3.0)
    want = O.brute(od, oq, O.RANGE, radii=np.full(4, 3.0))
    c, i, d = csr(got)
    assert np.array_equal(i, want.ids) and np.array_equal(d, want.dis)


@pytest.mark.parametrize("name", ["snap_words", "snap_l2"])
def test_snapshot_loaded_index_matches_brute(name):
    """A reference-written GTSI snapshot (tests/golden, io.py:60-89) drives the
    device index directly (stored tree, tombstones included)."""
    import os
    tree = P.load_snapshot(os.path.join(os.path.dirname(__file__), "golden", name + ".gtsi"))
    ds = tree.dataset
    rng = np.random.default_rng(9)
    dead = np.zeros(ds.n, np.uint8)
    dead[tree.rows[tree.tombstone == 1]] = 1
    if ds.metric == P.EDIT:
        q = string_queries(ds.strings, 20, rng, "abcdefghijz")
        od, oq = O.Payloads.from_strings(ds.strings, ids=ds.ids), O.Payloads.from_strings(q)
        radii = rng.integers(0, 5, 20).astype(float)
    else:
        q = list(f32(ds.mat[rng.integers(0, ds.n, 20)] + rng.normal(0, 0.02, (20, ds.dim))))
        od, oq = O.Payloads(O.L2, vec=ds.mat, ids=ds.ids), O.Payloads(O.L2, vec=np.array(q))
        radii = rng.uniform(0.05, 0.4, 20)
    ks = rng.integers(1, 25, 20)
    eng = P.BatchSearcher(tree)
    ans, _ = eng.range_batch(q, radii)
    c, i, d = csr(ans)
    want = O.brute(od, oq, O.RANGE, radii=radii, dead_rows=dead)
    assert np.array_equal(i, want.ids) and np.array_equal(d, want.dis)
    ans, _ = eng.knn_batch(q, ks)
    c, i, d = csr(ans)
    want = O.brute(od, oq, O.KNN, ks=ks, dead_rows=dead)
    assert np.array_equal(i, want.ids) and np.array_equal(d, want.dis)
