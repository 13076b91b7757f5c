"""GTSI snapshots (reference io.py:25-150): files written
by the reference's save_snapshot load into the drop-in FlatPivotTree, and
save_snapshot here reproduces them byte for byte."""

import os

import numpy as np
import pytest

import paper_2404_00966_b200 as P

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("name", ["snap_words", "snap_l2"])
def test_snapshot_roundtrip_bytes(name, tmp_path):
    src = os.path.join(GOLDEN, name + ".gtsi")
    tree = P.load_snapshot(src)
    assert tree.node_count > 0 and tree.rows.size == tree.dataset.n
    # the table covers every object once
    assert np.array_equal(np.sort(tree.rows), np.arange(tree.dataset.n))
    out = tmp_path / "again.gtsi"
    P.save_snapshot(tree, str(out))
    assert open(src, "rb").read() == open(out, "rb").read()


def test_snapshot_errors(tmp_path):
    bad = tmp_path / "bad.gtsi"
    bad.write_bytes(b"NOPE" + bytes(60))
    with pytest.raises(P.SnapshotFormatError):
        P.load_snapshot(str(bad))
    data = open(os.path.join(GOLDEN, "snap_l2.gtsi"), "rb").read()
    bad.write_bytes(data[:-3])
    with pytest.raises(P.SnapshotFormatError):
        P.load_snapshot(str(bad))
    bad.write_bytes(data + b"x")
    with pytest.raises(P.SnapshotFormatError):
        P.load_snapshot(str(bad))
