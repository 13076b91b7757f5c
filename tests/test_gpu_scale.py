"""Bench-scale parity and the buffer grow / re-run paths.

* 1M-object indexes (the words and 128-d bench shapes, BASELINE.json
  configs[1] / configs[2]): a full batch runs on the device (radius
  dynamics, chunking and buffer sizes of the real workload) and a sample of
  its queries is compared with oracle brute force.
* Small initial hit / candidate buffers (GTS_HIT_CAP0, GTS_CAND_CAP0) and an
  early kNN hit compaction (GTS_COMPACT_AT) force every grow-and-re-run path
  (engine.cu Search::verify, with_candidates, compact_hits) at test sizes.
"""

import numpy as np
import pytest

import paper_2404_00966_b200 as P
from oracle import oracle as O
from test_gpu_parity import check_against_oracle, csr, f32, string_queries

pytestmark = pytest.mark.gpu


def sample_matches(eng, queries, radii, ks, od, oq_of, sample):
    ans, _ = eng.range_batch(queries, radii)
    got = [ans[i] for i in sample]
    want = O.brute(od, oq_of([queries[i] for i in sample]), O.RANGE, radii=radii[sample], threads=16).answers()
    for g, w in zip(got, want):
        assert np.array_equal(g[0], w[0]) and np.array_equal(g[1], w[1])
    ans, _ = eng.knn_batch(queries, ks)
    got = [ans[i] for i in sample]
    want = O.brute(od, oq_of([queries[i] for i in sample]), O.KNN, ks=ks[sample], threads=16).answers()
    for g, w in zip(got, want):
        assert np.array_equal(g[0], w[0]) and np.array_equal(g[1], w[1])


def test_words_1m_batch_10k():
    rng = np.random.default_rng(51)
    alpha = "abcdefghijklmnopqrstuvwxyz"
    strs = P.generate_sequences(1_000_000, seed=52, min_len=1, max_len=34, alphabet=alpha)
    tree = P.build(P.Dataset.from_strings(strs, P.EDIT), P.TreeConfig(20, 0))
    q = string_queries(strs, 10_000, rng, alpha)
    sample = rng.choice(10_000, 48, replace=False)
    sample_matches(P.BatchSearcher(tree), q, np.full(10_000, 1.0), np.full(10_000, 10),
                   O.Payloads.from_strings(strs), O.Payloads.from_strings, sample)


def test_l2_128d_1m_batch_20k():
    rng = np.random.default_rng(53)
    mat = f32(P.generate_clustered(1_000_000, 128, 1000, seed=54, spread=0.05))
    tree = P.build(P.Dataset.from_vectors(mat, P.L2), P.TreeConfig(20, 0))
    q = f32(mat[rng.integers(0, 1_000_000, 20_000)] + rng.normal(0, 0.01, (20_000, 128)))
    sample = rng.choice(20_000, 48, replace=False)
    sample_matches(P.BatchSearcher(tree), list(q), np.full(20_000, 0.5), np.full(20_000, 10),
                   O.Payloads(O.L2, vec=mat), lambda qs: O.Payloads(O.L2, vec=np.array(qs)), sample)


@pytest.mark.parametrize("kind", ["words", "l2_128", "l1_32", "l2_2"])
def test_buffer_grow_and_rerun_paths(kind, monkeypatch):
    monkeypatch.setenv("GTS_HIT_CAP0", "64")
    monkeypatch.setenv("GTS_CAND_CAP0", "64")
    monkeypatch.setenv("GTS_COMPACT_AT", "512")
    rng = np.random.default_rng(55)
    if kind == "words":
        alpha = "abcdefghijklmnop"
        strs = P.generate_sequences(30_000, seed=56, min_len=1, max_len=20, alphabet=alpha)
        ds = P.Dataset.from_strings(strs, P.EDIT)
        q = string_queries(strs, 200, rng, alpha)
        od, oq = O.Payloads.from_strings(strs), O.Payloads.from_strings(q)
        radii = rng.integers(0, 5, 200).astype(float)
    else:
        D, met, code = {"l2_128": (128, P.L2, O.L2), "l1_32": (32, P.L1, O.L1), "l2_2": (2, P.L2, O.L2)}[kind]
        mat = f32(P.generate_clustered(30_000, D, 20, seed=57, spread=0.05))
        ds = P.Dataset.from_vectors(mat, met)
        qv = f32(mat[rng.integers(0, 30_000, 200)] + rng.normal(0, 0.01, (200, D)))
        q = list(qv)
        od, oq = O.Payloads(code, vec=mat), O.Payloads(code, vec=qv)
        scale = {"l2_128": 0.8, "l1_32": 2.0, "l2_2": 0.05}[kind]
        radii = rng.uniform(0.2, 1.0, 200) * scale
    tree = P.build(ds, P.TreeConfig(20, 1))
    check_against_oracle(ds, tree, q, od, oq, radii, rng.integers(1, 80, 200), threads=16)


def test_l1_32d_2m_shard_batch_20k():
    # the L1 shard shape (configs[4] per GPU: spread 0.01, range r = 0.5, kNN k = 100)
    rng = np.random.default_rng(58)
    mat = f32(P.generate_clustered(2_000_000, 32, 1000, seed=59, spread=0.01))
    tree = P.build(P.Dataset.from_vectors(mat, P.L1), P.TreeConfig(20, 0))
    q = f32(mat[rng.integers(0, 2_000_000, 20_000)] + rng.normal(0, 0.005, (20_000, 32)))
    sample = rng.choice(20_000, 48, replace=False)
    sample_matches(P.BatchSearcher(tree), list(q), np.full(20_000, 0.5), np.full(20_000, 100),
                   O.Payloads(O.L1, vec=mat), lambda qs: O.Payloads(O.L1, vec=np.array(qs)), sample)


def test_dna_108_1m_batch_2k():
    # configs[3] shape (range r = 8, kNN k = 10); the brute-force check of a
    # 108 x 108 DP per pair over 1M objects keeps the sample small
    rng = np.random.default_rng(60)
    strs = P.generate_sequences(1_000_000, seed=61, min_len=108, max_len=108, alphabet="ACGT")
    tree = P.build(P.Dataset.from_strings(strs, P.EDIT), P.TreeConfig(20, 0))
    q = string_queries(strs, 2_000, rng, "ACGT")
    sample = rng.choice(2_000, 6, replace=False)
    sample_matches(P.BatchSearcher(tree), q, np.full(2_000, 8.0), np.full(2_000, 10),
                   O.Payloads.from_strings(strs), O.Payloads.from_strings, sample)


def test_float_collect_orders_ties_below_float32():
    # distances equal in float32 but not in float64, larger for smaller rows:
    # the (float32, row) sort puts them in row order and the tie fix-up
    # (k_fix_f32_ties) must restore (float64 distance, id) order
    N = 3000
    mat = np.zeros((N, 2))
    mat[:, 0] = 1.0 + (N - np.arange(N)) * 2.0 ** -40
    mat = np.concatenate([mat, np.random.default_rng(62).uniform(3, 4, (5000, 2))])
    ds = P.Dataset.from_vectors(mat, P.L2)
    tree = P.build(ds, P.TreeConfig(8, 0))
    q = [np.zeros(2), np.array([0.0, 1e-9])]
    check_against_oracle(ds, tree, q, O.Payloads(O.L2, vec=mat), O.Payloads(O.L2, vec=np.array(q)),
                         np.array([2.0, 1.5]), np.array([N // 2, 7]), threads=8)
