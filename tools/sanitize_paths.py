"""Small invocations of every device kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck) on the GPU box:

    compute-sanitizer --tool memcheck python tools/sanitize_paths.py

Each case runs range + kNN through the drop-in BatchSearcher on a few
thousand objects and checks the answers against brute force (oracle), so
a sanitizer run also proves the instrumented kernels still answer right.
Covers: k_root / k_expand / k_expand_grouped / k_probe* / k_leaf_edit /
k_leafgroup_edit / k_leafgroup_mma2 / k_leafgroup_tile / k_leafgroup_vec /
k_verify / k_recheck / collect, device build, in-place inserts, the
pending cache scan, and the sharded merge kernels.
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2404_00966_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402


def check(answers, want, what):
    for i, (got, w) in enumerate(zip(answers, want)):
        if not (np.array_equal(got[0], w[0]) and np.allclose(got[1], w[1], rtol=1e-12, atol=0)):
            raise SystemExit(f"{what}: query {i} differs")


def run_vec(metric, n, dim, env=None, clustered=False):
    for k in ("GTS_NO_GROUPED", "GTS_VEC_ROWWARP", "GTS_EDIT_GROUPED"):
        os.environ.pop(k, None)
    os.environ.update(env or {})
    rng = np.random.default_rng(dim)
    if clustered:
        cent = rng.random((20, dim))
        mat = cent[rng.integers(0, 20, n)] + 0.05 * rng.standard_normal((n, dim))
    else:
        mat = rng.random((n, dim))
    mat = mat.astype(np.float32).astype(np.float64)
    met = {1: P.L1, 2: P.L2}[metric]
    tree = P.build(P.Dataset.from_vectors(mat, met), P.TreeConfig(20, 0))
    q = mat[rng.integers(0, n, 24)] + 0.01
    eng = P.BatchSearcher(tree)
    r = float(np.median(np.abs(mat[:50, None, :] - mat[None, :50, :]).sum(-1) if metric == 1 else
                        np.sqrt(((mat[:50, None, :] - mat[None, :50, :]) ** 2).sum(-1)))) * 0.3
    rng_ans, _ = eng.range_batch(list(q), r)
    knn_ans, _ = eng.knn_batch(list(q), 10)
    od, oq = O.Payloads(metric, vec=mat), O.Payloads(metric, vec=q)
    check(rng_ans, O.brute(od, oq, O.RANGE, radii=np.full(len(q), r)).answers(), f"range {metric}/{dim} {env}")
    check(knn_ans, O.brute(od, oq, O.KNN, ks=np.full(len(q), 10)).answers(), f"knn {metric}/{dim} {env}")


def run_edit(env=None, alphabet="abcdefghijklmnopqrstuvwxyz", lo=1, hi=34, n=3000):
    for k in ("GTS_NO_GROUPED", "GTS_VEC_ROWWARP", "GTS_EDIT_GROUPED"):
        os.environ.pop(k, None)
    os.environ.update(env or {})
    strs = P.generate_sequences(n, seed=3, min_len=lo, max_len=hi, alphabet=alphabet)
    tree = P.build(P.Dataset.from_strings(strs, P.EDIT), P.TreeConfig(20, 0))
    rng = np.random.default_rng(4)
    q = [strs[int(i)] for i in rng.integers(0, n, 24)]
    eng = P.BatchSearcher(tree)
    rr = 2.0 if hi < 50 else 10.0
    rng_ans, _ = eng.range_batch(q, rr)
    knn_ans, _ = eng.knn_batch(q, 10)
    od, oq = O.Payloads.from_strings(strs), O.Payloads.from_strings(q)
    check(rng_ans, O.brute(od, oq, O.RANGE, radii=np.full(len(q), rr)).answers(), f"edit range {env}")
    check(knn_ans, O.brute(od, oq, O.KNN, ks=np.full(len(q), 10)).answers(), f"edit knn {env}")


def run_stream():
    strs = P.generate_sequences(2000, seed=5, min_len=5, max_len=20, alphabet="ACGT")
    idx = P.StreamingIndex(P.Dataset.from_strings(strs, P.EDIT), P.TreeConfig(20, 0), cache_capacity=64)
    live = dict(enumerate(strs))
    for i in range(40):
        idx.delete(i)
        del live[i]
        idx.insert(5000 + i, strs[i + 100][::-1])
        live[5000 + i] = strs[i + 100][::-1]
    q = [strs[7], strs[300], strs[1500]]
    ans = idx.query_knn(q, 5)
    ans = ans[0] if isinstance(ans, tuple) else ans
    ids = np.array(sorted(live), dtype=np.int64)
    od = O.Payloads.from_strings([live[i] for i in ids])
    want = O.brute(od, O.Payloads.from_strings(q), O.KNN, ks=np.full(3, 5)).answers()
    for got, w in zip(ans, want):
        if not (np.array_equal(got[0], ids[w[0]]) and np.array_equal(got[1], w[1])):
            raise SystemExit("stream knn differs")


def main():
    cases = sys.argv[1:] or ["edit", "edit_grouped", "dna", "l2_2d", "l2_128", "l1_32", "rowwise", "rowwarp",
                             "stream"]
    for c in cases:
        if c == "edit":
            run_edit()
        elif c == "edit_grouped":
            run_edit({"GTS_EDIT_GROUPED": "1"})
        elif c == "dna":
            run_edit(alphabet="ACGT", lo=100, hi=108, n=1500)
        elif c == "l2_2d":
            run_vec(2, 4000, 2)
        elif c == "l2_128":
            run_vec(2, 3000, 128, clustered=True)
        elif c == "l1_32":
            run_vec(1, 3000, 32, clustered=True)
        elif c == "rowwise":
            run_vec(2, 2000, 32, {"GTS_NO_GROUPED": "1"})
        elif c == "rowwarp":
            run_vec(1, 2000, 16, {"GTS_VEC_ROWWARP": "1"})
        elif c == "stream":
            run_stream()
        print(f"ok {c}", flush=True)


if __name__ == "__main__":
    main()
