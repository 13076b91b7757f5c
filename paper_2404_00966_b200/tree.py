"""Flat pivot tree: arithmetic addressing, host build, device residency.

Mirrors reference tree.py (TreeConfig 40-57, tree_height 60-78, addressing
81-135, FlatPivotTree 138-215, build 370-385).  `build` runs the native
builder in libgts.so (csrc/builder.cpp); the device list tables are made
lazily by `FlatPivotTree.device_index()` (csrc/engine.cu gts_index_create).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .metrics import METRIC_CODES, STRING_METRICS

ROOT_ID = 1


class ConfigError(ValueError):
    """Invalid index configuration."""


class OrdinalError(ValueError):
    """Child ordinal or node ordinal out of range."""


class EncodeRangeError(ValueError):
    """Distance outside [0, level_max] passed to the key encoder."""


@dataclass(frozen=True)
class TreeConfig:
    node_capacity: int = 20
    seed: int = 0
    store_leaf_only: bool = True

    def __post_init__(self):
        if self.node_capacity < 2:
            raise ConfigError("node_capacity must be >= 2")


def tree_height(n, nc):
    """(max_h, split_rounds) with integer arithmetic (tree.py:60-78)."""
    if nc < 2:
        raise ConfigError("node_capacity must be >= 2")
    if n < 1:
        raise ValueError("tree_height requires n >= 1")
    t, power = 0, 1
    while power < n + 1:
        power *= nc
        t += 1
    return t - 1, max(t - 2, 0)


def child_node_id(i, j, nc):
    if not 1 <= j <= nc:
        raise OrdinalError(f"child ordinal {j} outside [1, {nc}]")
    if i < 1:
        raise OrdinalError(f"node id {i} outside the tree")
    return (i - 1) * nc + j + 1


def parent_node_id(i, nc):
    if i < 2:
        raise OrdinalError("the root has no parent")
    return (i - 2) // nc + 1


def level_range(level, nc):
    if level < 1:
        raise OrdinalError("levels are numbered from 1")
    count = nc ** (level - 1)
    return (count - 1) // (nc - 1) + 1, count


def node_count_for(levels, nc):
    return (nc ** levels - 1) // (nc - 1)


def encode_distance(dis, ordinal, level_max):
    if ordinal < 0:
        raise OrdinalError("node ordinal must be >= 0")
    if not 0.0 <= dis <= level_max:
        raise EncodeRangeError(f"distance {dis} outside [0, {level_max}]")
    return dis / (level_max + 1.0) + ordinal


def decode_distance(key, ordinal, level_max):
    return (key - ordinal) * (level_max + 1.0)


class FlatPivotTree:
    """Node SoA + object table (reference layout: int64 / float64 arrays)."""

    def __init__(self, config, dataset):
        self.config = config
        self.dataset = dataset
        self.levels = 0
        self.max_h = 0
        self.split_rounds = 0
        n = dataset.n
        self.rows = np.arange(n, dtype=np.int64)
        self.dis = np.zeros(n, dtype=np.float64)
        self.tombstone = np.zeros(n, dtype=np.uint8)
        self._alloc_nodes(0)
        self._entry_pos = None
        self._dev = None
        self._dev_tomb = None

    def _alloc_nodes(self, count):
        self.pivot_id = np.full(count + 1, -1, dtype=np.int64)
        self.pivot_row = np.full(count + 1, -1, dtype=np.int64)
        self.min_dis = np.zeros(count + 1, dtype=np.float64)
        self.max_dis = np.zeros(count + 1, dtype=np.float64)
        self.pos = np.zeros(count + 1, dtype=np.int64)
        self.size = np.zeros(count + 1, dtype=np.int64)

    @property
    def n(self):
        return self.rows.size

    @property
    def node_count(self):
        return self.pivot_id.size - 1

    @property
    def nc(self):
        return self.config.node_capacity

    @property
    def object_ids(self):
        return self.dataset.ids[self.rows]

    def segment(self, node):
        p = self.pos[node]
        return self.rows[p: p + self.size[node]]

    def entry_pos_of_id(self, obj_id):
        if self._entry_pos is None:
            inv = np.empty(self.n, dtype=np.int64)
            inv[self.rows] = np.arange(self.n, dtype=np.int64)
            self._entry_pos = inv
        row = int(self.dataset.rows_of_ids([obj_id])[0])
        return int(self._entry_pos[row])

    # -- C-ABI views ---------------------------------------------------------

    def _c_tree(self):
        p = _lib.ptr
        return _lib.GtsTree(
            self.nc, self.levels, self.split_rounds, self.node_count, self.n,
            p(self.pivot_id, _lib._i64p), p(self.pivot_row, _lib._i64p), p(self.pos, _lib._i64p),
            p(self.size, _lib._i64p), p(self.min_dis, _lib._f64p), p(self.max_dis, _lib._f64p),
            p(self.rows, _lib._i64p), p(self.dis, _lib._f64p), p(self.tombstone, _lib._u8p))

    def device_index(self, device=0):
        """The device-resident list tables of this tree on `device` (created
        once per device; tombstones re-synced when they changed)."""
        if self._dev is None:
            self._dev, self._dev_tomb = {}, {}
        dev = self._dev.get(int(device))
        if dev is None:
            ds, keep = _c_dataset(self.dataset)
            h = C.c_void_p()
            t = self._c_tree()
            _lib.check(_lib.lib().gts_index_create(C.byref(ds), C.byref(t), int(device), C.byref(h)))
            dev = self._dev[int(device)] = _DeviceIndex(h)
            self._dev_tomb[int(device)] = self.tombstone.copy()
        elif not np.array_equal(self._dev_tomb[int(device)], self.tombstone):
            tomb = np.ascontiguousarray(self.tombstone, dtype=np.uint8)
            _lib.check(_lib.lib().gts_index_set_tombstones(dev.h, _lib.ptr(tomb, _lib._u8p), None))
            self._dev_tomb[int(device)] = tomb.copy()
        return dev


class _DeviceIndex:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            if self.h:
                _lib.lib().gts_index_destroy(self.h)
                self.h = None
        except Exception:
            pass


def _c_dataset(ds):
    """C view of a Dataset; returns (struct, arrays-to-keep-alive)."""
    p = _lib.ptr
    ids = np.ascontiguousarray(ds.ids, dtype=np.int64)
    if ds.metric in STRING_METRICS:
        codes = ds.codes if ds.codes.size else np.zeros(1, np.int32)
        s = _lib.GtsDataset(METRIC_CODES[ds.metric], ds.n, 0, None, p(codes, _lib._i32p),
                            p(ds.offsets, _lib._i64p), p(ids, _lib._i64p))
        return s, (codes, ids)
    mat = np.ascontiguousarray(ds.mat, dtype=np.float64)
    s = _lib.GtsDataset(METRIC_CODES[ds.metric], ds.n, ds.dim, p(mat, _lib._f64p), None, None, p(ids, _lib._i64p))
    return s, (mat, ids)


def build(dataset, config=None, runtime=None, threads=0, device=None):
    """Build a FlatPivotTree (tree.py:370-385) with the native builder:
    host C++/OpenMP by default, or on GPU `device` (gts_build_tree_device;
    edit / l1 / l2, the same tree bit for bit)."""
    config = config or TreeConfig()
    tree = FlatPivotTree(config, dataset)
    n = dataset.n
    if n == 0:
        return tree
    nc = config.node_capacity
    tree.max_h, tree.split_rounds = tree_height(n, nc)
    tree.levels = tree.split_rounds + 1
    tree._alloc_nodes(node_count_for(tree.levels, nc))
    # the reference's root draw (tree.py:263, 288-291)
    root_row = int(np.random.default_rng(config.seed).integers(0, n))
    ds, keep = _c_dataset(dataset)
    t = tree._c_tree()
    if device is None:
        _lib.check(_lib.lib().gts_build_tree(C.byref(ds), root_row, int(threads), C.byref(t)))
    else:
        _lib.check(_lib.lib().gts_build_tree_device(C.byref(ds), root_row, int(device), C.byref(t)))
    return tree
