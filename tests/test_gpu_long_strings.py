"""Edit-distance queries longer than 32 * kMaxWords = 4096 symbols.

The reference DP (metrics.py:54-84) has no length limit.  Patterns beyond
4096 symbols run the row-band bit-parallel DP (kernels.cuh myers_banded);
answers must equal the oracle's brute force exactly.  A pair whose both
sides exceed 4096 symbols is refused with ValueError (GTS_EINVAL)."""

import numpy as np
import pytest

import paper_2404_00966_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _strings(n, lo, hi, seed, alphabet="ACGT"):
    rng = np.random.default_rng(seed)
    return ["".join(rng.choice(list(alphabet), size=int(rng.integers(lo, hi + 1)))) for _ in range(n)]


def test_queries_longer_than_4096_symbols():
    base = _strings(400, 200, 900, seed=1)
    rng = np.random.default_rng(2)
    # long queries: stored strings repeated / mutated into 4.1k-9k symbols
    queries = []
    for i in range(6):
        s = "".join(base[int(j)] for j in rng.integers(0, 400, 12))
        s = (s * 2)[: int(rng.integers(4100, 9000))]
        queries.append(s)
    queries.append(base[3] + "A" * 4200)          # shares a prefix with an indexed string
    queries.append(base[5][:100])                  # an ordinary short query in the same batch
    tree = P.build(P.Dataset.from_strings(base, P.EDIT), P.TreeConfig(20, 0))
    eng = P.BatchSearcher(tree)
    od, oq = O.Payloads.from_strings(base), O.Payloads.from_strings(queries)
    radii = np.array([max(len(q) - 150.0, 60.0) for q in queries])
    got, _ = eng.range_batch(queries, radii)
    want = O.brute(od, oq, O.RANGE, radii=radii, threads=8).answers()
    for g, w in zip(got, want):
        assert np.array_equal(g[0], w[0]) and np.array_equal(g[1], w[1])
    got, _ = eng.knn_batch(queries, 5)
    want = O.brute(od, oq, O.KNN, ks=np.full(len(queries), 5), threads=8).answers()
    for g, w in zip(got, want):
        assert np.array_equal(g[1], w[1])
        assert np.array_equal(g[0], w[0])


def test_both_sides_longer_than_4096_refused():
    base = _strings(30, 4200, 4300, seed=3)
    tree = P.build(P.Dataset.from_strings(base, P.EDIT), P.TreeConfig(20, 0))
    with pytest.raises(ValueError):
        P.BatchSearcher(tree).range_batch([base[0] + "A"], 10.0)
