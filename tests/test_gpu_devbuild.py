"""Device bulk build (gts_build_tree_device, csrc/devbuild.cuh; SURVEY.md
§8(f1)) against the reference's own trees (tests/golden, made by the
unmodified reference) and against the host builder on larger seeded
collections: every tree array must be bit-identical (tree.py:241-385)."""

import ctypes as C

import numpy as np
import pytest
import torch

import paper_2404_00966_b200 as P
from paper_2404_00966_b200 import _lib
from paper_2404_00966_b200.tree import node_count_for
from conftest import TREES, load_golden
from test_host import TREE_FIELDS, dataset_of

pytestmark = pytest.mark.gpu


def same_tree(a, b):
    assert a.levels == b.levels and a.split_rounds == b.split_rounds
    for f in TREE_FIELDS:
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


@pytest.mark.parametrize("name", TREES)
def test_device_build_matches_reference_tree(name):
    g = load_golden(name)
    t = P.build(dataset_of(g), P.TreeConfig(int(g["nc"]), int(g["seed"])), device=0)
    assert t.levels == int(g["levels"]) and t.split_rounds == int(g["split_rounds"])
    for f in TREE_FIELDS:
        assert np.array_equal(getattr(t, f), g[f]), f


def _collections():
    rng = np.random.default_rng(5)
    yield "words", P.Dataset.from_strings(P.generate_sequences(60000, seed=1, min_len=1, max_len=34,
                                                               alphabet="abcdefghijklmnopqrstuvwxyz"), P.EDIT)
    yield "dna", P.Dataset.from_strings(P.generate_sequences(6000, seed=2, min_len=108, max_len=108,
                                                             alphabet="ACGT"), P.EDIT)
    yield "long", P.Dataset.from_strings(P.generate_sequences(800, seed=3, min_len=0, max_len=300,
                                                              alphabet="ab"), P.EDIT)
    yield "l2_2d", P.Dataset.from_vectors(rng.uniform(0, 1, (200000, 2)), P.L2)
    yield "l1_32d", P.Dataset.from_vectors(rng.uniform(0, 1, (60000, 32)).astype(np.float32), P.L1)
    yield "grid", P.Dataset.from_vectors(np.round(rng.uniform(0, 6, (30000, 3))), P.L1,
                                         ids=np.arange(30000) * 7 + 3)
    yield "l2_128d", P.Dataset.from_vectors(rng.normal(0, 1, (20000, 128)), P.L2)


@pytest.mark.parametrize("nc", [20, 3])
def test_device_build_matches_host_builder(nc):
    for name, ds in _collections():
        same_tree(P.build(ds, P.TreeConfig(nc, 4), device=0), P.build(ds, P.TreeConfig(nc, 4)))


def test_device_build_f32_entry_point():
    """Device-resident float32 input (the generator's output) builds the same
    tree as the float64 host path over the widened values."""
    rng = np.random.default_rng(9)
    x = rng.uniform(0, 1, (50000, 32)).astype(np.float32)
    ds = P.Dataset.from_vectors(x.astype(np.float64), P.L1)
    want = P.build(ds, P.TreeConfig(20, 0))
    dx = torch.from_numpy(x).cuda()
    got = P.FlatPivotTree(P.TreeConfig(20, 0), ds)
    got.max_h, got.split_rounds = P.tree_height(ds.n, 20)
    got.levels = got.split_rounds + 1
    got._alloc_nodes(node_count_for(got.levels, 20))
    t = got._c_tree()
    root = int(np.random.default_rng(0).integers(0, ds.n))
    _lib.check(_lib.lib().gts_build_tree_device_f32(1, ds.n, 32, C.c_void_p(dx.data_ptr()),
                                                    _lib.ptr(ds.ids, _lib._i64p), root, 0, C.byref(t)))
    same_tree(got, want)
