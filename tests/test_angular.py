"""Angular metric (reference metrics.py:136-193).

Angular distances cannot be pinned bit-exactly: numpy's arccos is a SIMD
implementation (not libm's acos) and the reference's query norm comes from
np.dot (BLAS, summation order unspecified).  Parity is therefore the north
star's float tolerance, applied far tighter than its 1e-5: tree structure
identical, ids identical, distances within 1e-12 relative / 1e-14 absolute.
CPU: the C oracle against fixtures produced by the reference itself.
GPU (test_gpu_angular.py): the device path against the oracle.
"""

import numpy as np
import pytest

from conftest import decode_strings, load_golden  # noqa: F401
from oracle import oracle as O

ANG = 3
REL, ABS = 1e-12, 1e-14


def close(a, b):
    return a.shape == b.shape and np.allclose(a, b, rtol=REL, atol=ABS)


def test_oracle_angular_pairs():
    m = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "metrics_angular.npz"))
    for k in m.files:
        if k.endswith("_d"):
            base = k[:-2]
            a, b = m[base + "_a"], m[base + "_b"]
            got = np.array([O.vec(ANG, a[i], b[i]) for i in range(len(a))])
            assert close(got, m[k]), k
            # the zero-vector / identical rules are exact
            exact = (m[k] == 0.0) | (m[k] == np.pi)
            assert np.array_equal(got[exact], m[k][exact]), k


def test_oracle_angular_tree_and_search():
    g = load_golden("angular_16d")
    data = O.Payloads(ANG, vec=g["data_vec"], ids=g["ids"])
    qs = O.Payloads(ANG, vec=g["query_vec"])
    t = O.build(data, int(g["nc"]), int(g["seed"]))
    for f in ["pivot_id", "pivot_row", "pos", "size", "rows"]:
        assert np.array_equal(getattr(t, f), g[f]), f
    for f in ["min_dis", "max_dis", "dis"]:
        assert close(getattr(t, f), g[f]), f
    for mode, kind in ((O.RANGE, "range"), (O.KNN, "knn")):
        r = O.search(t, data, qs, mode, radii=g["radii"], ks=g["ks"])
        k = f"{kind}_wide"
        assert np.array_equal(r.counts, g[k + "_counts"])
        assert np.array_equal(r.ids, g[k + "_ids"])
        assert close(r.dis, g[k + "_dis"])
