"""ctypes front end of the CPU oracle (oracle/gts_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / `--impl reference` legs, never by the product
package.  It restates the reference `metrictree` build + BatchSearcher +
brute force (see the C header for file:line citations) and is pinned
against tests/golden/*.npz, which were produced by the reference itself.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

EDIT, L1, L2 = 0, 1, 2
RANGE, KNN = 0, 1
_MAX_LAYERS = 64

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)


class _Ds(C.Structure):
    _fields_ = [
        ("metric", C.c_int64), ("n", C.c_int64), ("dim", C.c_int64),
        ("vec", _f64p), ("codes", _i32p), ("off", _i64p), ("ids", _i64p),
    ]


class _Tree(C.Structure):
    _fields_ = [
        ("nc", C.c_int64), ("levels", C.c_int64), ("split_rounds", C.c_int64),
        ("nodes", C.c_int64), ("n", C.c_int64),
        ("pivot_id", _i64p), ("pivot_row", _i64p), ("pos", _i64p), ("size", _i64p),
        ("min_dis", _f64p), ("max_dis", _f64p),
        ("rows", _i64p), ("dis", _f64p), ("tomb", _u8p),
    ]


class _Res(C.Structure):
    _fields_ = [
        ("nq", C.c_int64), ("counts", _i64p), ("ids", _i64p), ("dis", _f64p),
        ("total", C.c_int64), ("verified", _i64p), ("pruned", _i64p),
        ("peak", C.c_int64), ("limits", C.c_int64 * _MAX_LAYERS),
        ("status", C.c_int), ("err", C.c_char * 256),
    ]


def build_lib() -> str:
    """Compile liboracle.so (make in oracle/)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build_lib()
        L = C.CDLL(LIB_PATH)
        L.orc_search.restype = C.POINTER(_Res)
        L.orc_search.argtypes = [C.POINTER(_Tree), C.POINTER(_Ds), C.POINTER(_Ds), C.c_int,
                                 _f64p, _i64p, C.c_int64, C.c_int, C.c_int]
        L.orc_brute.restype = C.POINTER(_Res)
        L.orc_brute.argtypes = [C.POINTER(_Ds), _u8p, C.POINTER(_Ds), C.c_int, _f64p, _i64p, C.c_int]
        L.orc_result_free.argtypes = [C.POINTER(_Res)]
        L.orc_build.argtypes = [C.POINTER(_Ds), C.POINTER(_Tree), C.c_int64, C.c_int]
        L.orc_build.restype = C.c_int
        L.orc_tree_height.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p]
        L.orc_node_count.argtypes = [C.c_int64, C.c_int64]
        L.orc_node_count.restype = C.c_int64
        L.orc_edit.argtypes = [_i32p, C.c_int64, _i32p, C.c_int64]
        L.orc_edit.restype = C.c_double
        L.orc_vec.argtypes = [C.c_int64, _f64p, _f64p, C.c_int64]
        L.orc_vec.restype = C.c_double
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


class Payloads:
    """Dataset / query batch in the oracle's layout (keeps arrays alive)."""

    def __init__(self, metric, vec=None, codes=None, off=None, ids=None):
        self.metric = int(metric)
        if metric == EDIT:
            self.codes = np.ascontiguousarray(codes, dtype=np.int32)
            if self.codes.size == 0:
                self.codes = np.zeros(1, dtype=np.int32)
            self.off = np.ascontiguousarray(off, dtype=np.int64)
            self.n = self.off.size - 1
            self.dim = 0
            self.vec = np.zeros(1)
        else:
            self.vec = np.ascontiguousarray(vec, dtype=np.float64)
            self.n, self.dim = self.vec.shape
            self.codes = np.zeros(1, dtype=np.int32)
            self.off = np.zeros(1, dtype=np.int64)
        self.ids = np.ascontiguousarray(
            np.arange(self.n, dtype=np.int64) if ids is None else ids, dtype=np.int64)
        self.s = _Ds(self.metric, self.n, self.dim, _p(self.vec, _f64p), _p(self.codes, _i32p),
                     _p(self.off, _i64p), _p(self.ids, _i64p))

    @staticmethod
    def from_strings(strings, ids=None):
        lens = np.array([len(s) for s in strings], dtype=np.int64)
        off = np.zeros(len(strings) + 1, dtype=np.int64)
        np.cumsum(lens, out=off[1:])
        codes = (np.frombuffer("".join(strings).encode("utf-32-le"), dtype=np.int32)
                 if strings else np.empty(0, np.int32))
        return Payloads(EDIT, codes=codes, off=off, ids=ids)


class Tree:
    """Flat pivot tree arrays (reference tree.py:155-175 layout, int64/f64)."""

    def __init__(self, nc, levels, split_rounds, pivot_id, pivot_row, min_dis, max_dis,
                 pos, size, rows, dis, tombstone=None):
        self.nc, self.levels, self.split_rounds = int(nc), int(levels), int(split_rounds)
        c = np.ascontiguousarray
        self.pivot_id = c(pivot_id, dtype=np.int64)
        self.pivot_row = c(pivot_row, dtype=np.int64)
        self.min_dis = c(min_dis, dtype=np.float64)
        self.max_dis = c(max_dis, dtype=np.float64)
        self.pos = c(pos, dtype=np.int64)
        self.size = c(size, dtype=np.int64)
        self.rows = c(rows, dtype=np.int64)
        self.dis = c(dis, dtype=np.float64)
        self.tombstone = (np.zeros(self.rows.size, dtype=np.uint8) if tombstone is None
                          else c(tombstone, dtype=np.uint8))
        self._sync()

    def _sync(self):
        self.s = _Tree(self.nc, self.levels, self.split_rounds, self.pivot_id.size - 1, self.rows.size,
                       _p(self.pivot_id, _i64p), _p(self.pivot_row, _i64p), _p(self.pos, _i64p),
                       _p(self.size, _i64p), _p(self.min_dis, _f64p), _p(self.max_dis, _f64p),
                       _p(self.rows, _i64p), _p(self.dis, _f64p),
                       _p(self.tombstone if self.tombstone.size else np.zeros(1, np.uint8), _u8p))


def tree_height(n, nc):
    mh, sp = C.c_int64(), C.c_int64()
    lib().orc_tree_height(n, nc, C.byref(mh), C.byref(sp))
    return mh.value, sp.value


def root_row(n, seed):
    """The reference's root draw: default_rng(seed).integers(0, n) (tree.py:263, 289)."""
    return int(np.random.default_rng(seed).integers(0, n))


def build(data: Payloads, nc: int, seed: int, threads: int = 0) -> Tree:
    """Restated reference build (tree.py:370-385)."""
    n = data.n
    if n == 0:
        z = np.zeros(1)
        return Tree(nc, 0, 0, np.full(1, -1), np.full(1, -1), z, z, np.zeros(1), np.zeros(1),
                    np.zeros(0), np.zeros(0))
    _, split = tree_height(n, nc)
    levels = split + 1
    nodes = lib().orc_node_count(levels, nc)
    t = Tree(nc, levels, split, np.full(nodes + 1, -1), np.full(nodes + 1, -1), np.zeros(nodes + 1),
             np.zeros(nodes + 1), np.zeros(nodes + 1), np.zeros(nodes + 1), np.zeros(n), np.zeros(n))
    rc = lib().orc_build(C.byref(data.s), C.byref(t.s), root_row(n, seed), int(threads))
    if rc:
        raise RuntimeError("orc_build failed")
    return t


class Result:
    def __init__(self, ptr):
        r = ptr.contents
        nq = r.nq
        self.counts = np.ctypeslib.as_array(r.counts, (nq,)).copy() if nq else np.zeros(0, np.int64)
        tot = r.total
        self.ids = np.ctypeslib.as_array(r.ids, (tot,)).copy() if tot else np.zeros(0, np.int64)
        self.dis = np.ctypeslib.as_array(r.dis, (tot,)).copy() if tot else np.zeros(0)
        self.verified = np.ctypeslib.as_array(r.verified, (nq,)).copy() if nq else np.zeros(0, np.int64)
        self.pruned = np.ctypeslib.as_array(r.pruned, (nq,)).copy() if nq else np.zeros(0, np.int64)
        self.peak = int(r.peak)
        self.size_limits = {l: int(r.limits[l]) for l in range(_MAX_LAYERS) if r.limits[l]}
        self.status = int(r.status)
        self.err = r.err.decode()
        lib().orc_result_free(ptr)
        self.offsets = np.zeros(nq + 1, dtype=np.int64)
        np.cumsum(self.counts, out=self.offsets[1:])

    def answers(self):
        return [(self.ids[self.offsets[q]:self.offsets[q + 1]], self.dis[self.offsets[q]:self.offsets[q + 1]])
                for q in range(self.counts.size)]


def search(tree: Tree, data: Payloads, queries: Payloads, mode, radii=None, ks=None,
           memory_units=1 << 20, pruning=True, threads=1) -> Result:
    """Restated BatchSearcher.range_batch / knn_batch (search.py:238-296)."""
    nq = queries.n
    radii = np.ascontiguousarray(np.broadcast_to(np.asarray(0.0 if radii is None else radii, np.float64), (nq,)))
    ks = np.ascontiguousarray(np.broadcast_to(np.asarray(1 if ks is None else ks, np.int64), (nq,)))
    tree._sync()
    ptr = lib().orc_search(C.byref(tree.s), C.byref(data.s), C.byref(queries.s), int(mode),
                           _p(radii, _f64p), _p(ks, _i64p), int(memory_units), int(bool(pruning)),
                           int(threads))
    return Result(ptr)


def brute(data: Payloads, queries: Payloads, mode, radii=None, ks=None, dead_rows=None, threads=1) -> Result:
    """Restated oracle.brute_range / brute_knn (oracle.py:19-47)."""
    nq = queries.n
    radii = np.ascontiguousarray(np.broadcast_to(np.asarray(0.0 if radii is None else radii, np.float64), (nq,)))
    ks = np.ascontiguousarray(np.broadcast_to(np.asarray(1 if ks is None else ks, np.int64), (nq,)))
    dead = None
    if dead_rows is not None:
        dead = np.ascontiguousarray(dead_rows, dtype=np.uint8)
    ptr = lib().orc_brute(C.byref(data.s), None if dead is None else _p(dead, _u8p), C.byref(queries.s),
                          int(mode), _p(radii, _f64p), _p(ks, _i64p), int(threads))
    return Result(ptr)


def edit(a: str, b: str) -> float:
    ca = np.frombuffer(a.encode("utf-32-le"), dtype=np.int32).copy() if a else np.zeros(1, np.int32)
    cb = np.frombuffer(b.encode("utf-32-le"), dtype=np.int32).copy() if b else np.zeros(1, np.int32)
    return lib().orc_edit(_p(ca, _i32p), len(a), _p(cb, _i32p), len(b))


def vec(metric, x, q) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    return lib().orc_vec(int(metric), _p(x, _f64p), _p(q, _f64p), x.size)
