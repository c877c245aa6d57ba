"""Host-side value types mirroring the reference package's public types.

Same names, fields, conventions and validation as the reference
(/root/reference/pkg/src/sparse_kmeans), so code written against
``sparse_kmeans`` reads the same against this package:

* ``Dataset``     <- data.py:130-227   (CSR, 1-based int32 terms, float64 values)
* ``MeanSet``     <- means.py:24-188   (mean-major CSR + representation tag)
* ``Assignment``  <- variants.py:37-70 (1-based labels + sizes, FNV-1a digest)
* ``OpCounters``  <- counters.py:22-44
* ``CorruptionError`` <- data.py:27-28

Reference objects are accepted wherever these are (duck-typed on the same
attributes).  Heavy work never happens here: these types only validate and
carry arrays between the caller and the device engine.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property

import numpy as np

__all__ = [
    "CorruptionError", "Dataset", "MeanSet", "Assignment", "OpCounters", "COUNTER_FIELDS",
    "REPRESENTATIONS", "fnv1a64",
]

_NORM_TOL = 1e-12
REPRESENTATIONS = ("dense", "dense_inverted", "sparse_inverted", "sparse_standard")
COUNTER_FIELDS = ("mults", "adds", "inner_entries", "branch_checks", "merge_steps")


class CorruptionError(RuntimeError):
    """An id inside a postings list points outside its owner range (data.py:27-28)."""


def _frozen(a: np.ndarray) -> np.ndarray:
    a.setflags(write=False)
    return a


def _rows_strictly_increasing(arr: np.ndarray, indptr: np.ndarray) -> bool:
    """data.py:36-43."""
    if arr.size < 2:
        return True
    inner = np.ones(arr.size, dtype=bool)
    starts = indptr[1:-1]
    inner[starts[starts < arr.size]] = False
    return not np.any((np.diff(arr) <= 0) & inner[1:])


def _row_sq_norms(indptr: np.ndarray, values: np.ndarray) -> np.ndarray:
    """Per-row sum of squares (validation only: the 1e-12 unit-norm check)."""
    n = indptr.size - 1
    out = np.zeros(n)
    if values.size == 0 or n == 0:
        return out
    nonempty = indptr[1:] > indptr[:-1]
    out[nonempty] = np.add.reduceat(values * values, indptr[:-1][nonempty])
    return out


@dataclass(frozen=True, eq=False)
class Dataset:
    """Objects in CSR layout (data.py:130-227): row i holds term_ids[indptr[i]:indptr[i+1]]
    (1-based, strictly increasing) and float64 values; ``normalized`` asserts unit rows."""

    dim: int
    indptr: np.ndarray
    term_ids: np.ndarray
    values: np.ndarray
    normalized: bool = False
    dropped_docs: tuple = ()

    def __post_init__(self):
        ip = np.ascontiguousarray(self.indptr, dtype=np.int64)
        t = np.ascontiguousarray(self.term_ids, dtype=np.int32)
        v = np.ascontiguousarray(self.values, dtype=np.float64)
        if ip.ndim != 1 or ip.size < 1 or ip[0] != 0 or ip[-1] != t.size:
            raise ValueError("malformed indptr")
        if np.any(np.diff(ip) < 0):
            raise ValueError("indptr must be non-decreasing")
        if t.shape != v.shape:
            raise ValueError("term_ids and values must be parallel")
        if t.size:
            if t.min() < 1 or t.max() > self.dim:
                raise ValueError("term ids must lie in 1..dim")
            if not _rows_strictly_increasing(t, ip):
                raise ValueError("term ids must be strictly increasing per row")
        if not np.all(np.isfinite(v)) or np.any(v == 0.0):
            raise ValueError("values must be finite and nonzero")
        if self.normalized and ip.size > 1:
            if np.any(np.abs(np.sqrt(_row_sq_norms(ip, v)) - 1.0) > _NORM_TOL):
                raise ValueError("normalized dataset has a non-unit row")
        object.__setattr__(self, "indptr", _frozen(ip))
        object.__setattr__(self, "term_ids", _frozen(t))
        object.__setattr__(self, "values", _frozen(v))

    @property
    def n(self) -> int:
        return int(self.indptr.size - 1)

    @property
    def sum_nnz(self) -> int:
        return int(self.term_ids.size)

    @cached_property
    def nnz_per_doc(self) -> np.ndarray:
        return _frozen(np.diff(self.indptr))

    @cached_property
    def doc_freq(self) -> np.ndarray:
        """data.py:208-211: slot p-1 counts term p."""
        return _frozen(np.bincount(self.term_ids, minlength=self.dim + 1)[1:])


@dataclass(frozen=True, eq=False)
class MeanSet:
    """k unit-norm means as a mean-major CSR (means.py:24-64)."""

    k: int
    dim: int
    representation: str
    indptr: np.ndarray
    term_ids: np.ndarray
    values: np.ndarray
    retained: np.ndarray

    def __post_init__(self):
        if self.representation not in REPRESENTATIONS:
            raise ValueError(f"unknown representation {self.representation!r}")
        ip = np.ascontiguousarray(self.indptr, dtype=np.int64)
        t = np.ascontiguousarray(self.term_ids, dtype=np.int32)
        v = np.ascontiguousarray(self.values, dtype=np.float64)
        r = np.ascontiguousarray(self.retained, dtype=bool)
        if ip.size != self.k + 1 or ip[0] != 0 or ip[-1] != t.size:
            raise ValueError("malformed indptr")
        if r.size != self.k:
            raise ValueError("retained flags must have length k")
        if t.size and (t.min() < 1 or t.max() > self.dim):
            raise ValueError("term ids must lie in 1..dim")
        if not _rows_strictly_increasing(t, ip):
            raise ValueError("term ids must be strictly increasing per mean")
        if np.any(np.abs(np.sqrt(_row_sq_norms(ip, v)) - 1.0) > _NORM_TOL):
            raise ValueError("every mean must have unit L2 norm")
        object.__setattr__(self, "indptr", _frozen(ip))
        object.__setattr__(self, "term_ids", _frozen(t))
        object.__setattr__(self, "values", _frozen(v))
        object.__setattr__(self, "retained", _frozen(r))

    @classmethod
    def trusted(cls, k, dim, representation, indptr, term_ids, values, retained) -> "MeanSet":
        """Wrap arrays produced by the device update without re-validating them:
        its output is strictly increasing per mean and unit-norm by
        construction (bit-identical to variants.py:254-307, whose MeanSet the
        tests validate).  Arrays are frozen, not copied."""
        obj = cls.__new__(cls)
        for name, val in (("k", int(k)), ("dim", int(dim)), ("representation", representation),
                          ("indptr", indptr), ("term_ids", term_ids), ("values", values),
                          ("retained", retained)):
            if isinstance(val, np.ndarray):
                val.setflags(write=False)
            object.__setattr__(obj, name, val)
        return obj

    @classmethod
    def from_csr(cls, indptr, term_ids, values, dim, representation="sparse_standard",
                 retained=None) -> "MeanSet":
        k = int(np.asarray(indptr).size - 1)
        if retained is None:
            retained = np.zeros(k, dtype=bool)
        return cls(k, dim, representation, indptr, term_ids, values, retained)

    def with_representation(self, representation: str) -> "MeanSet":
        if representation == self.representation:
            return self
        return MeanSet(self.k, self.dim, representation, self.indptr, self.term_ids,
                       self.values, self.retained)

    @cached_property
    def term_counts(self) -> np.ndarray:
        return _frozen(np.diff(self.indptr))

    @cached_property
    def centroid_freq(self) -> np.ndarray:
        """means.py:144-147: (nc)_p, slot p-1 holds term p."""
        return _frozen(np.bincount(self.term_ids, minlength=self.dim + 1)[1:])

    @property
    def sum_terms(self) -> int:
        return int(self.term_ids.size)


@dataclass(frozen=True, eq=False)
class Assignment:
    """1-based labels and per-cluster sizes (variants.py:37-70)."""

    labels: np.ndarray
    sizes: np.ndarray

    def __post_init__(self):
        labels = np.ascontiguousarray(self.labels, dtype=np.int32)
        sizes = np.ascontiguousarray(self.sizes, dtype=np.int64)
        if labels.size and (labels.min() < 1 or labels.max() > sizes.size):
            raise ValueError("labels must lie in 1..k")
        if int(sizes.sum()) != labels.size:
            raise ValueError("sizes must sum to the number of objects")
        labels.setflags(write=False)
        sizes.setflags(write=False)
        object.__setattr__(self, "labels", labels)
        object.__setattr__(self, "sizes", sizes)

    @classmethod
    def from_labels(cls, labels: np.ndarray, k: int) -> "Assignment":
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        return cls(labels, np.bincount(labels - 1, minlength=k).astype(np.int64))

    @property
    def n(self) -> int:
        return int(self.labels.size)

    @property
    def k(self) -> int:
        return int(self.sizes.size)

    def digest(self) -> int:
        return fnv1a64(self.labels.astype("<i4", copy=False))


@dataclass
class OpCounters:
    """counters.py:25-44."""

    mults: int = 0
    adds: int = 0
    inner_entries: int = 0
    branch_checks: int = 0
    merge_steps: int = 0

    @classmethod
    def from_array(cls, arr) -> "OpCounters":
        return cls(*(int(x) for x in arr))

    def to_dict(self) -> dict:
        return {name: getattr(self, name) for name in COUNTER_FIELDS}

    def add_array(self, arr) -> None:
        for name, x in zip(COUNTER_FIELDS, arr):
            setattr(self, name, getattr(self, name) + int(x))


def fnv1a64(data) -> int:
    """64-bit FNV-1a (variants.py:77-83) over raw bytes or a contiguous array's
    bytes, computed by the native library."""
    import ctypes

    from . import _lib

    fn = _lib.load().ivfkm_fnv1a64
    if isinstance(data, np.ndarray):
        arr = np.ascontiguousarray(data)
        return int(fn(ctypes.c_void_p(arr.ctypes.data), arr.nbytes))
    data = bytes(data)
    return int(fn(ctypes.cast(ctypes.c_char_p(data), ctypes.c_void_p), len(data)))
