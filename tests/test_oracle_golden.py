"""The CPU oracle (oracle/) against fixtures produced by the reference itself."""

import numpy as np
import pytest

from conftest import TIGHT_UNITS, TREES, load_golden
from oracle import oracle as O

TREE_FIELDS = ["pivot_id", "pivot_row", "min_dis", "max_dis", "pos", "size", "rows", "dis"]


def payloads(g):
    met = int(g["metric"])
    if met == 0:
        return (O.Payloads(0, codes=g["data_codes"], off=g["data_off"], ids=g["ids"]),
                O.Payloads(0, codes=g["query_codes"], off=g["query_off"]))
    return O.Payloads(met, vec=g["data_vec"], ids=g["ids"]), O.Payloads(met, vec=g["query_vec"])


def test_oracle_metrics(golden_metrics):
    m = golden_metrics
    ao, bo, ac, bc = m["edit_a_off"], m["edit_b_off"], m["edit_a_codes"], m["edit_b_codes"]
    for i in range(m["edit_d"].size):
        a = "".join(map(chr, ac[ao[i]:ao[i + 1]]))
        b = "".join(map(chr, bc[bo[i]:bo[i + 1]]))
        assert O.edit(a, b) == m["edit_d"][i]
    for k in m.files:
        if k.startswith("vec") and k.endswith("_l1"):
            base = k[:-3]
            a, b = m[base + "_a"], m[base + "_b"]
            for met, key in ((O.L1, "_l1"), (O.L2, "_l2")):
                got = np.array([O.vec(met, a[i], b[i]) for i in range(len(a))])
                assert np.array_equal(got, m[base + key]), base + key  # bit-exact


@pytest.mark.parametrize("name", TREES)
def test_oracle_tree_and_search(name):
    g = load_golden(name)
    data, qs = payloads(g)
    t = O.build(data, int(g["nc"]), int(g["seed"]))
    for f in TREE_FIELDS:
        assert np.array_equal(getattr(t, f), g[f]), f
    runs = [("", None, "wide", 1 << 20), ("", None, "tight", TIGHT_UNITS[name]),
            ("dead_", g["tombstone"], "wide", 1 << 20)]
    for prefix, tomb, tag, units in runs:
        t.tombstone = np.zeros(t.rows.size, np.uint8) if tomb is None else tomb.copy()
        for mode, kind in ((O.RANGE, "range"), (O.KNN, "knn")):
            r = O.search(t, data, qs, mode, radii=g["radii"], ks=g["ks"], memory_units=units)
            k = f"{prefix}{kind}_{tag}"
            assert np.array_equal(r.counts, g[k + "_counts"])
            assert np.array_equal(r.ids, g[k + "_ids"])
            assert np.array_equal(r.dis, g[k + "_dis"])
            assert np.array_equal(r.verified, g[k + "_verified"])
            assert np.array_equal(r.pruned, g[k + "_pruned"])
            assert r.peak == int(g[k + "_peak"])
            if kind == "range" and prefix == "":
                lim = g[k + "_limits"]
                assert r.size_limits == {int(a): int(b) for a, b in lim}
    r = O.search(t, data, qs, O.RANGE, radii=g["radii"], pruning=False)
    assert np.array_equal(r.ids, g["dead_nopr_range_ids"])
    assert np.array_equal(r.verified, g["dead_nopr_range_verified"])
    dead = np.zeros(data.n, np.uint8)
    dead[t.rows[t.tombstone == 1]] = 1
    b = O.brute(data, qs, O.RANGE, radii=g["radii"], dead_rows=dead)
    assert np.array_equal(b.ids, g["dead_range_wide_ids"])
    assert np.array_equal(b.dis, g["dead_range_wide_dis"])
