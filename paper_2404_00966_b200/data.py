"""Datasets and synthetic generators (reference data.py:59-418).

Payloads stay on the host in the reference layout (float64 matrix, or
strings + packed int32 code points); the device copy in table order is
made by the index (csrc/engine.cu gts_index_create).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .metrics import (
    METRIC_KINDS,
    STRING_METRICS,
    VECTOR_METRICS,
    MetricMismatchError,
    as_vector,
    encode_string,
    pack_strings,
)

SEQUENCE_ALPHABET = "ACGTN"


@dataclass(frozen=True)
class DataObject:
    """One identified object (data.py:51-56)."""

    id: int
    payload: object


class Dataset:
    """Payloads under one metric with strictly increasing int64 ids (data.py:136-156)."""

    def __init__(self, metric, mat=None, strings=None, ids=None):
        if metric not in METRIC_KINDS:
            raise MetricMismatchError(f"unknown metric kind: {metric!r}")
        self.metric = metric
        if metric in VECTOR_METRICS:
            if mat is None:
                raise MetricMismatchError(f"metric {metric!r} requires vector payloads")
            mat = np.asarray(mat, dtype=np.float64)
            if mat.ndim != 2:
                raise MetricMismatchError("vector store requires a 2-D matrix")
            if not np.all(np.isfinite(mat)):
                raise MetricMismatchError("vector payloads contain non-finite values")
            self.mat = np.ascontiguousarray(mat)
            self.strings = None
            self.codes = self.offsets = None
            n = self.mat.shape[0]
        else:
            if strings is None:
                raise MetricMismatchError(f"metric {metric!r} requires string payloads")
            self.strings = list(strings)
            for s in self.strings:
                if not isinstance(s, str):
                    raise MetricMismatchError("string dataset requires str payloads")
            self.codes, self.offsets = pack_strings(self.strings)
            self.mat = None
            n = len(self.strings)
        ids = np.arange(n, dtype=np.int64) if ids is None else np.asarray(ids, dtype=np.int64)
        if ids.ndim != 1 or ids.size != n:
            raise ValueError("ids must be a 1-D array matching the payload count")
        if ids.size and (np.any(ids < 0) or np.any(np.diff(ids) <= 0)):
            raise ValueError("ids must be non-negative and strictly increasing")
        self.ids = ids

    @classmethod
    def from_vectors(cls, mat, metric, ids=None):
        mat = np.atleast_2d(np.asarray(mat, dtype=np.float64))
        return cls(metric, mat=mat, ids=ids)

    @classmethod
    def from_strings(cls, strings, metric, ids=None):
        return cls(metric, strings=list(strings), ids=ids)

    @classmethod
    def from_objects(cls, objects, metric):
        objs = sorted(objects, key=lambda o: o.id)
        ids = np.array([o.id for o in objs], dtype=np.int64)
        payloads = [o.payload for o in objs]
        if metric in VECTOR_METRICS:
            mat = np.asarray(payloads, dtype=np.float64) if payloads else np.empty((0, 0))
            return cls(metric, mat=np.atleast_2d(mat), ids=ids)
        return cls(metric, strings=payloads, ids=ids)

    @property
    def n(self):
        return self.mat.shape[0] if self.mat is not None else len(self.strings)

    def __len__(self):
        return self.n

    @property
    def dim(self):
        return self.mat.shape[1] if self.mat is not None else None

    def payload(self, row):
        return self.mat[row].copy() if self.mat is not None else self.strings[row]

    def object_at(self, row):
        return DataObject(int(self.ids[row]), self.payload(row))

    def rows_of_ids(self, wanted):
        wanted = np.asarray(wanted, dtype=np.int64)
        rows = np.searchsorted(self.ids, wanted)
        if np.any(rows >= self.ids.size) or np.any(self.ids[np.minimum(rows, self.ids.size - 1)] != wanted):
            raise KeyError("unknown object id")
        return rows

    def prepare_query(self, payload):
        """Encode / validate one query payload (data.py:220-229)."""
        if self.metric in STRING_METRICS:
            return encode_string(payload)
        v = as_vector(payload)
        if self.n and v.shape[0] != self.dim:
            raise MetricMismatchError(
                f"query dimensionality {v.shape[0]} != dataset dimensionality {self.dim}")
        return v

    def prepare_batch(self, payloads):
        """Validated batch in the C-ABI layout: (vectors f64 [nq, D]) or (codes, offsets)."""
        if self.metric in STRING_METRICS:
            for p in payloads:
                encode_string(p)
            return pack_strings(list(payloads))
        vs = [self.prepare_query(p) for p in payloads]
        if not vs:
            return np.zeros((0, self.dim or 0))
        return np.ascontiguousarray(np.stack(vs))

    def subset_rows(self, rows, ids=None):
        rows = np.asarray(rows, dtype=np.int64)
        ids = self.ids[rows] if ids is None else ids
        if self.mat is not None:
            return Dataset(self.metric, mat=self.mat[rows], ids=ids)
        return Dataset(self.metric, strings=[self.strings[r] for r in rows], ids=ids)


def generate_uniform(n, dim, seed, low=0.0, high=1.0):
    """Uniform vectors in [low, high)^dim (data.py:399-402)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(low, high, size=(n, dim))


def generate_clustered(n, dim, clusters, seed, spread=0.01, box=1.0):
    """Gaussian clusters (data.py:405-410)."""
    rng = np.random.default_rng(seed)
    centers = rng.uniform(0.0, box, size=(clusters, dim))
    assign = rng.integers(0, clusters, size=n)
    return centers[assign] + rng.normal(0.0, spread * box, size=(n, dim))


def generate_sequences(n, seed, min_len=4, max_len=40, alphabet=SEQUENCE_ALPHABET):
    """Random symbol strings, uniform lengths (data.py:413-418)."""
    rng = np.random.default_rng(seed)
    lengths = rng.integers(min_len, max_len + 1, size=n)
    syms = np.array(list(alphabet))
    return ["".join(syms[rng.integers(0, len(syms), size=l)]) for l in lengths]
