"""GTSI snapshots, byte-compatible with the reference (io.py:25-150; SURVEY.md
§8(f) f3): a snapshot written by `metrictree.save_snapshot` loads here into a
FlatPivotTree whose device index is built straight from the stored arrays (no
rebuild), and `save_snapshot` here writes the identical bytes.

Layout (little-endian, padding-free): header "<4sHBxqqqqqq" (magic GTSI,
version 1, metric code, seed, n, node_capacity, levels, split_rounds, max_h);
nodes [node_count] {pivot_id i8, min_dis f8, max_dis f8, pos i8, size i8};
table [n] {object_id i8, dis f8, tombstone u1}; ids [n] i8; payloads
(strings: offsets [n+1] i8 + UTF-8 blob; vectors: dim i8 + [n*dim] f8).
"""

from __future__ import annotations

import struct

import numpy as np

from .data import Dataset
from .metrics import METRIC_CODES, STRING_METRICS
from .tree import FlatPivotTree, TreeConfig, node_count_for

SNAPSHOT_MAGIC = b"GTSI"
SNAPSHOT_VERSION = 1
_HEADER = struct.Struct("<4sHBxqqqqqq")
_METRIC_NAMES = {v: k for k, v in METRIC_CODES.items()}
NODE_DTYPE = np.dtype([("pivot_id", "<i8"), ("min_dis", "<f8"), ("max_dis", "<f8"), ("pos", "<i8"), ("size", "<i8")])
TABLE_DTYPE = np.dtype([("object_id", "<i8"), ("dis", "<f8"), ("tombstone", "<u1")])


class SnapshotFormatError(ValueError):
    """Bad magic, unsupported version, or truncated snapshot (io.py:57-58)."""


def save_snapshot(tree, path):
    """Write a built index and its dataset (io.py:60-89)."""
    ds = tree.dataset
    node_count = tree.node_count
    header = _HEADER.pack(SNAPSHOT_MAGIC, SNAPSHOT_VERSION, METRIC_CODES[ds.metric], int(tree.config.seed),
                          int(ds.n), int(tree.config.node_capacity), int(tree.levels), int(tree.split_rounds),
                          int(tree.max_h))
    nodes = np.empty(node_count, dtype=NODE_DTYPE)
    if node_count:
        nodes["pivot_id"] = tree.pivot_id[1:]
        nodes["min_dis"] = tree.min_dis[1:]
        nodes["max_dis"] = tree.max_dis[1:]
        nodes["pos"] = tree.pos[1:]
        nodes["size"] = tree.size[1:]
    table = np.empty(ds.n, dtype=TABLE_DTYPE)
    table["object_id"] = tree.object_ids
    table["dis"] = tree.dis
    table["tombstone"] = tree.tombstone
    with open(path, "wb") as fh:
        fh.write(header)
        fh.write(nodes.tobytes())
        fh.write(table.tobytes())
        fh.write(ds.ids.astype("<i8").tobytes())
        if ds.metric in STRING_METRICS:
            blobs = [s.encode("utf-8") for s in ds.strings]
            offsets = np.zeros(len(blobs) + 1, dtype="<i8")
            np.cumsum([len(b) for b in blobs], out=offsets[1:])
            fh.write(offsets.tobytes())
            fh.write(b"".join(blobs))
        else:
            fh.write(struct.pack("<q", int(ds.dim if ds.n else 0)))
            fh.write(ds.mat.astype("<f8").tobytes())


def _take(buf, off, dtype, count):
    nbytes = dtype.itemsize * count
    if off + nbytes > len(buf):
        raise SnapshotFormatError("snapshot truncated")
    return np.frombuffer(buf, dtype=dtype, count=count, offset=off), off + nbytes


def load_snapshot(path):
    """Read a snapshot back into a FlatPivotTree, dataset included (io.py:106-150)."""
    with open(path, "rb") as fh:
        buf = fh.read()
    if len(buf) < _HEADER.size:
        raise SnapshotFormatError("snapshot truncated before header")
    magic, version, mcode, seed, n, nc, levels, split_rounds, max_h = _HEADER.unpack_from(buf, 0)
    if magic != SNAPSHOT_MAGIC:
        raise SnapshotFormatError(f"bad magic {magic!r}")
    if version != SNAPSHOT_VERSION:
        raise SnapshotFormatError(f"unsupported snapshot version {version}")
    if mcode not in _METRIC_NAMES:
        raise SnapshotFormatError(f"unknown metric code {mcode}")
    metric = _METRIC_NAMES[mcode]
    node_count = node_count_for(levels, nc) if levels > 0 else 0
    off = _HEADER.size
    nodes, off = _take(buf, off, NODE_DTYPE, node_count)
    table, off = _take(buf, off, TABLE_DTYPE, n)
    ids, off = _take(buf, off, np.dtype("<i8"), n)
    if metric in STRING_METRICS:
        offsets, off = _take(buf, off, np.dtype("<i8"), n + 1)
        blob_len = int(offsets[-1]) if n else 0
        if off + blob_len > len(buf):
            raise SnapshotFormatError("snapshot truncated in string payloads")
        blob = buf[off:off + blob_len]
        off += blob_len
        ds = Dataset.from_strings([blob[offsets[i]:offsets[i + 1]].decode("utf-8") for i in range(n)], metric,
                                  ids=ids.copy())
    else:
        if off + 8 > len(buf):
            raise SnapshotFormatError("snapshot truncated before vector header")
        (dim,) = struct.unpack_from("<q", buf, off)
        off += 8
        mat, off = _take(buf, off, np.dtype("<f8"), n * dim)
        ds = Dataset.from_vectors(mat.reshape(n, dim).copy(), metric, ids=ids.copy())
    if off != len(buf):
        raise SnapshotFormatError(f"{len(buf) - off} trailing bytes")
    tree = FlatPivotTree(TreeConfig(node_capacity=int(nc), seed=int(seed)), ds)
    tree.levels = int(levels)
    tree.split_rounds = int(split_rounds)
    tree.max_h = int(max_h)
    tree._alloc_nodes(node_count)
    if node_count:
        tree.pivot_id[1:] = nodes["pivot_id"]
        tree.min_dis[1:] = nodes["min_dis"]
        tree.max_dis[1:] = nodes["max_dis"]
        tree.pos[1:] = nodes["pos"]
        tree.size[1:] = nodes["size"]
        assigned = tree.pivot_id >= 0
        tree.pivot_row[assigned] = ds.rows_of_ids(tree.pivot_id[assigned])
    if n:
        tree.rows = ds.rows_of_ids(table["object_id"]).astype(np.int64)
        tree.dis = table["dis"].astype(np.float64)
        tree.tombstone = table["tombstone"].astype(np.uint8)
    return tree
