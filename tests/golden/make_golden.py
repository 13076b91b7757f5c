"""Generate golden fixtures by running the UNMODIFIED reference package.

Run in the build container only (it imports the read-only reference from
/root/reference/pkg/src, which does not exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Outputs `tests/golden/*.npz`, which the tests read at run time.  Every vector
payload is generated in float64, cast to float32 and widened back, so the
same values are exactly representable on the device (SURVEY.md finding 3).

Fixtures:
  metrics.npz  edit / L1 / L2 distances of random pairs (reference
               metrics.py:54-193), plus the known answers of
               test_metrics.py:41-56.
  tree_<name>.npz   FlatPivotTree arrays (reference tree.py:138-385) and
               BatchSearcher answers + SearchStats (search.py:214-570) for a
               range batch and a kNN batch, with default and tight budgets,
               and a tombstoned variant.
"""

from __future__ import annotations

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from metrictree import metrics  # noqa: E402
from metrictree.data import (  # noqa: E402
    Dataset,
    generate_clustered,
    generate_sequences,
    generate_uniform,
)
from metrictree.search import BatchSearcher  # noqa: E402
from metrictree.tree import TreeConfig, build  # noqa: E402

METRIC_CODE = {metrics.EDIT: 0, metrics.L1: 1, metrics.L2: 2, metrics.ANGULAR: 3}


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def pack_strings(strings):
    lens = np.array([len(s) for s in strings], dtype=np.int64)
    off = np.zeros(len(strings) + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    if strings:
        codes = np.frombuffer("".join(strings).encode("utf-32-le"), dtype=np.int32)
    else:
        codes = np.empty(0, dtype=np.int32)
    return codes.copy(), off


def csr(answers):
    counts = np.array([a[0].size for a in answers], dtype=np.int64)
    ids = np.concatenate([a[0] for a in answers]) if answers else np.empty(0, np.int64)
    dis = np.concatenate([a[1] for a in answers]) if answers else np.empty(0)
    return counts, ids.astype(np.int64), dis.astype(np.float64)


def gen_metrics():
    rng = np.random.default_rng(1234)
    out = {}
    # edit: random pairs over several alphabets and lengths (incl. > 64, > 128)
    sa, sb = [], []
    for t in range(600):
        alpha = ["ab", "ACGT", "abcdefghijklmnopqrstuvwxyz", "aé漢"][t % 4]
        la = int(rng.integers(0, 140 if t % 5 == 0 else 40))
        lb = int(rng.integers(0, 140 if t % 7 == 0 else 40))
        a = "".join(alpha[int(i)] for i in rng.integers(0, len(alpha), la))
        if t % 3 == 0 and la:
            # near-duplicate: a few edits of a
            b = list(a)
            for _ in range(int(rng.integers(0, 4))):
                if b and rng.integers(0, 2):
                    b[int(rng.integers(0, len(b)))] = alpha[int(rng.integers(0, len(alpha)))]
                else:
                    b.insert(int(rng.integers(0, len(b) + 1)), alpha[int(rng.integers(0, len(alpha)))])
            b = "".join(b)
        else:
            b = "".join(alpha[int(i)] for i in rng.integers(0, len(alpha), lb))
        sa.append(a)
        sb.append(b)
    known = [("kitten", "sitting"), ("flaw", "lawn"), ("", "abc"), ("abc", ""), ("", "")]
    sa += [k[0] for k in known]
    sb += [k[1] for k in known]
    ed = np.array([metrics.edit_distance(a, b) for a, b in zip(sa, sb)])
    out["edit_a_codes"], out["edit_a_off"] = pack_strings(sa)
    out["edit_b_codes"], out["edit_b_off"] = pack_strings(sb)
    out["edit_d"] = ed
    # vectors: L1/L2 per dimensionality, fp32-representable and raw f64
    for D in (1, 2, 3, 7, 8, 9, 16, 31, 32, 33, 100, 128, 129, 200, 300):
        a = rng.normal(size=(40, D)) * 3.0
        b = rng.normal(size=(40, D)) * 3.0
        for tag, (xa, xb) in (("f32", (f32(a), f32(b))), ("f64", (a, b))):
            out[f"vec_{tag}_{D}_a"] = xa
            out[f"vec_{tag}_{D}_b"] = xb
            out[f"vec_{tag}_{D}_l1"] = metrics.l1_row_pairs(xa, xb)
            out[f"vec_{tag}_{D}_l2"] = metrics.l2_row_pairs(xa, xb)
    out["known_l1"] = np.array([metrics.distance(metrics.L1, [0, 0], [3, 4])])
    out["known_l2"] = np.array([metrics.distance(metrics.L2, [0, 0], [3, 4])])
    np.savez_compressed(os.path.join(HERE, "metrics.npz"), **out)


def tree_arrays(tree):
    return {
        "levels": np.int64(tree.levels),
        "split_rounds": np.int64(tree.split_rounds),
        "pivot_id": tree.pivot_id.copy(),
        "pivot_row": tree.pivot_row.copy(),
        "min_dis": tree.min_dis.copy(),
        "max_dis": tree.max_dis.copy(),
        "pos": tree.pos.copy(),
        "size": tree.size.copy(),
        "rows": tree.rows.copy(),
        "dis": tree.dis.copy(),
    }


def run_searches(tree, queries, radii, ks, prefix, out, budgets):
    for tag, units in budgets:
        eng = BatchSearcher(tree, memory_units=units)
        ans, st = eng.range_batch(queries, radii)
        c, i, d = csr(ans)
        out[f"{prefix}range_{tag}_counts"] = c
        out[f"{prefix}range_{tag}_ids"] = i
        out[f"{prefix}range_{tag}_dis"] = d
        out[f"{prefix}range_{tag}_verified"] = st.verified.copy()
        out[f"{prefix}range_{tag}_pruned"] = st.pruned_nodes.copy()
        out[f"{prefix}range_{tag}_peak"] = np.int64(st.peak_units)
        out[f"{prefix}range_{tag}_limits"] = np.array(sorted(st.size_limits.items()), dtype=np.int64).reshape(-1, 2)
        ans, st = eng.knn_batch(queries, ks)
        c, i, d = csr(ans)
        out[f"{prefix}knn_{tag}_counts"] = c
        out[f"{prefix}knn_{tag}_ids"] = i
        out[f"{prefix}knn_{tag}_dis"] = d
        out[f"{prefix}knn_{tag}_verified"] = st.verified.copy()
        out[f"{prefix}knn_{tag}_pruned"] = st.pruned_nodes.copy()
        out[f"{prefix}knn_{tag}_peak"] = np.int64(st.peak_units)


def gen_tree(name, ds, nc, seed, queries, radii, ks, tight_units, dead_frac=0.2):
    out = {"metric": np.int64(METRIC_CODE[ds.metric]), "nc": np.int64(nc), "seed": np.int64(seed)}
    if ds.metric == metrics.EDIT:
        out["data_codes"], out["data_off"] = pack_strings(ds.store.strings)
        out["query_codes"], out["query_off"] = pack_strings(queries)
    else:
        out["data_vec"] = ds.store.mat.copy()
        out["query_vec"] = np.array(queries, dtype=np.float64).reshape(len(queries), -1)
    out["ids"] = ds.ids.copy()
    tree = build(ds, TreeConfig(node_capacity=nc, seed=seed))
    out.update(tree_arrays(tree))
    out["radii"] = np.asarray(radii, dtype=np.float64)
    out["ks"] = np.asarray(ks, dtype=np.int64)
    run_searches(tree, queries, radii, ks, "", out, [("wide", None), ("tight", tight_units)])
    # tombstoned variant (same tree object, marks applied in place)
    rng = np.random.default_rng(seed + 99)
    dead = rng.choice(ds.n, int(ds.n * dead_frac), replace=False)
    dead_ids = ds.ids[np.sort(dead)]
    for oid in dead_ids:
        tree.tombstone[tree.entry_pos_of_id(int(oid))] = 1
    out["dead_ids"] = dead_ids
    out["tombstone"] = tree.tombstone.copy()
    run_searches(tree, queries, radii, ks, "dead_", out, [("wide", None)])
    # pruning disabled
    eng = BatchSearcher(tree, pruning=False)
    ans, st = eng.range_batch(queries, radii)
    c, i, d = csr(ans)
    out["dead_nopr_range_counts"], out["dead_nopr_range_ids"], out["dead_nopr_range_dis"] = c, i, d
    out["dead_nopr_range_verified"] = st.verified.copy()
    np.savez_compressed(os.path.join(HERE, f"tree_{name}.npz"), **out)
    print(name, "n", ds.n, "levels", tree.levels, "nodes", tree.node_count)


def vector_queries(mat, nq, rng):
    members = [mat[int(i)].copy() for i in rng.integers(0, mat.shape[0], nq // 2)]
    lo, hi = mat.min(axis=0), mat.max(axis=0)
    fresh = [f32(rng.uniform(lo, hi)) for _ in range(nq - nq // 2)]
    return members + fresh


def string_queries(strings, nq, rng):
    members = [strings[int(i)] for i in rng.integers(0, len(strings), nq // 2)]
    alphabet = sorted({c for s in strings[:200] for c in s}) or ["a"]
    mutated = []
    for i in rng.integers(0, len(strings), nq - nq // 2):
        s = list(strings[int(i)])
        for _ in range(int(rng.integers(1, 3))):
            c = alphabet[int(rng.integers(0, len(alphabet)))]
            if s and rng.integers(0, 2):
                s[int(rng.integers(0, len(s)))] = c
            else:
                s.insert(int(rng.integers(0, len(s) + 1)), c)
        mutated.append("".join(s))
    return members + mutated


def gen_trees():
    rng = np.random.default_rng(7)
    # 10-point line, nc=2, seed 0 (test_tree.py:209-215)
    line = np.arange(10, dtype=np.float64)[:, None]
    ds = Dataset.from_vectors(line, metrics.L2)
    gen_tree("line10", ds, 2, 0, [line[3], line[7]], [1.5, 0.0], [3, 4], 8)
    # 2-D L2 uniform (T-Loc-like), n=3000, nc=8
    mat = f32(generate_uniform(3000, 2, seed=12))
    ds = Dataset.from_vectors(mat, metrics.L2)
    q = vector_queries(mat, 64, rng)
    gen_tree("l2_2d", ds, 8, 1, q, rng.uniform(0.0, 0.08, 64), rng.integers(1, 24, 64), 64)
    # L1 integer grid (tie heavy), 4-D, n=2000, nc=5
    mat = np.round(generate_uniform(2000, 4, seed=11) * 20)
    ds = Dataset.from_vectors(mat, metrics.L1)
    q = vector_queries(mat, 48, rng)
    q = [np.round(x) for x in q]
    gen_tree("l1_grid", ds, 5, 2, q, rng.integers(0, 12, 48).astype(float), rng.integers(1, 32, 48), 40)
    # 32-d L1 clustered, n=2000, nc=6
    mat = f32(generate_clustered(2000, 32, 20, seed=5, spread=0.05))
    ds = Dataset.from_vectors(mat, metrics.L1)
    q = vector_queries(mat, 32, rng)
    gen_tree("l1_32d", ds, 6, 3, q, rng.uniform(0.5, 3.0, 32), rng.integers(1, 40, 32), 60)
    # 128-d L2 clustered, n=1500, nc=4
    mat = f32(generate_clustered(1500, 128, 15, seed=6, spread=0.05))
    ds = Dataset.from_vectors(mat, metrics.L2)
    q = vector_queries(mat, 24, rng)
    gen_tree("l2_128d", ds, 4, 4, q, rng.uniform(0.2, 1.0, 24), rng.integers(1, 16, 24), 16)
    # edit: ACGTN sequences (reference generator defaults), n=1500, nc=3
    strs = generate_sequences(1500, seed=14)
    ds = Dataset.from_strings(strs, metrics.EDIT)
    q = string_queries(strs, 40, rng)
    gen_tree("edit_seq", ds, 3, 5, q, rng.integers(0, 9, 40).astype(float), rng.integers(1, 20, 40), 30)
    # edit: words-like a-z len 1..34, n=9000, nc=20 (C2 shape, small)
    strs = generate_sequences(9000, seed=21, min_len=1, max_len=34, alphabet="abcdefghijklmnopqrstuvwxyz")
    ds = Dataset.from_strings(strs, metrics.EDIT)
    q = string_queries(strs, 40, rng)
    gen_tree("edit_words", ds, 20, 6, q, rng.integers(0, 4, 40).astype(float), rng.integers(1, 12, 40), 100)
    # edit: DNA len 108 (C4 shape, small), n=600, nc=4
    strs = generate_sequences(600, seed=22, min_len=108, max_len=108, alphabet="ACGT")
    ds = Dataset.from_strings(strs, metrics.EDIT)
    q = string_queries(strs, 16, rng)
    gen_tree("edit_dna", ds, 4, 7, q, rng.integers(0, 60, 16).astype(float), rng.integers(1, 10, 16), 20)


def gen_angular():
    """Angular fixtures (metrics.py:136-193), generated separately so the
    fixtures above stay byte-identical: pair distances incl. the zero-vector
    and exact-equality rules, and one 16-d clustered tree with zero vectors
    and duplicates."""
    rng = np.random.default_rng(4321)
    out = {}
    for D in (2, 3, 16, 33, 128):
        a = f32(rng.normal(size=(60, D)))
        b = f32(rng.normal(size=(60, D)))
        b[:6] = a[:6]                          # identical -> 0
        b[6:10] = a[6:10] * 2.0                # parallel -> ~0 (not identical)
        a[10:12] = 0.0                         # zero vs non-zero -> pi
        a[12:14] = 0.0
        b[12:14] = 0.0                         # zero vs zero -> 0
        b[14:16] = -a[14:16]                   # antiparallel -> pi
        na = np.sqrt((a * a).sum(axis=1))
        nb = np.sqrt((b * b).sum(axis=1))
        out[f"ang_{D}_a"], out[f"ang_{D}_b"] = a, b
        out[f"ang_{D}_d"] = metrics.angular_row_pairs(a, b, na, nb)
    np.savez_compressed(os.path.join(HERE, "metrics_angular.npz"), **out)
    # 16-d clustered tree with zero rows and duplicates
    mat = f32(generate_clustered(1500, 16, 12, seed=31, spread=0.08) - 0.5)
    mat[:5] = 0.0
    mat[5:15] = mat[100:110]
    ds = Dataset.from_vectors(mat, metrics.ANGULAR)
    q = vector_queries(mat, 40, rng)
    q[0] = np.zeros(16)
    q[1] = mat[7].copy()
    gen_tree("angular_16d", ds, 5, 8, q, rng.uniform(0.0, 0.6, 40), rng.integers(1, 30, 40), 40)


def gen_snapshots():
    """GTSI snapshots written by the reference's save_snapshot (io.py:60-89):
    a words tree with tombstones and an angular / L2 vector tree."""
    from metrictree.io import save_snapshot
    strs = generate_sequences(800, seed=41, min_len=1, max_len=20, alphabet="abcdefghij") + ["", "é漢"]
    ids = np.arange(len(strs), dtype=np.int64) * 3 + 5          # non-contiguous ids
    tree = build(Dataset.from_strings(strs, metrics.EDIT, ids=ids), TreeConfig(node_capacity=6, seed=3))
    for oid in ids[::17]:
        tree.tombstone[tree.entry_pos_of_id(int(oid))] = 1
    save_snapshot(tree, os.path.join(HERE, "snap_words.gtsi"))
    mat = f32(generate_clustered(700, 12, 7, seed=42, spread=0.1))
    tree = build(Dataset.from_vectors(mat, metrics.L2), TreeConfig(node_capacity=5, seed=4))
    save_snapshot(tree, os.path.join(HERE, "snap_l2.gtsi"))


if __name__ == "__main__":
    if "--angular" in sys.argv:
        gen_angular()
    elif "--snapshots" in sys.argv:
        gen_snapshots()
    else:
        gen_metrics()
        gen_trees()
        gen_angular()
        gen_snapshots()
