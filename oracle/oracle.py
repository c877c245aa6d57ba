"""ORACLE — test infrastructure only (tests/, __graft_entry__.smoke(), bench.py's
cpu_baseline and --impl reference legs).  The product package never imports it.

CPU restatement of the reference IVF Lloyd path, each function citing the
reference file:line it follows (paths under /root/reference/pkg/src/sparse_kmeans):

* assign      -> oracle/ivf_oracle.c (C restatement of _kernels.pyx:106-128), or the
                 reference's own compiled kernel in oracle/_ref when it was built
                 here (oracle/build_ref.sh), loaded by ``ref_kernels()``
* inverted    -> means.py:169-179   MeanSet.inverted
* update      -> variants.py:240-307 _member_entry_order + update_means
* objective   -> clustering.py:105-119 objective_cosine (the reference's dense k x D
                 gather when it fits in memory, else the same products gathered
                 from the sparse CSR; same per-object order, fsum)
* volume      -> counters.py:71-81  mult_volume_ivf
* seeding     -> clustering.py:41-102 SplitMix64 / sample_without_replacement / init_means
* run         -> clustering.py:229-315 (IVF branch)
* fnv1a64     -> variants.py:77-83

Pinned by tests/test_oracle.py against the reference's hand-computed answers
and against golden vectors produced by running the reference itself
(tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes as C
import importlib.util
import math
import os
import subprocess
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
BUILD = HERE / "_build"
LIB = BUILD / "liboracle.so"
REF_DIR = HERE / "_ref"


# ---------------------------------------------------------------- C oracle

def build(force: bool = False) -> Path:
    src = HERE / "ivf_oracle.c"
    if force or not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        BUILD.mkdir(exist_ok=True)
        subprocess.run(["gcc", "-O3", "-ffp-contract=off", "-fPIC", "-shared", "-pthread",
                        "-o", str(LIB), str(src)], check=True)
    return LIB


_c = None


def clib():
    global _c
    if _c is None:
        build()
        lib = C.CDLL(str(LIB))
        lib.oracle_assign_ivf.restype = C.c_int
        lib.oracle_assign_ivf.argtypes = [C.c_int64] + [C.c_void_p] * 6 + [C.c_int64] + \
            [C.c_void_p] * 4 + [C.c_int]
        lib.oracle_fnv1a64.restype = C.c_uint64
        lib.oracle_fnv1a64.argtypes = [C.c_void_p, C.c_size_t]
        _c = lib
    return _c


def _vp(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def assign_ivf(indptr, terms, vals, m_indptr, m_cids, m_vals, k, threads=1):
    """C restatement of _kernels.pyx:106-128 (+ top-two similarities).

    Returns (labels 1-based int32, top1 float64, top2 float64, postings touched).
    """
    ip = np.ascontiguousarray(indptr, np.int64)
    t = np.ascontiguousarray(terms, np.int32)
    v = np.ascontiguousarray(vals, np.float64)
    mp = np.ascontiguousarray(m_indptr, np.int64)
    mc = np.ascontiguousarray(m_cids, np.int32)
    mv = np.ascontiguousarray(m_vals, np.float64)
    n = ip.size - 1
    labels = np.empty(n, np.int32)
    top1 = np.empty(n, np.float64)
    top2 = np.empty(n, np.float64)
    ctr = np.zeros(5, np.int64)
    rc = clib().oracle_assign_ivf(n, _vp(ip), _vp(t), _vp(v), _vp(mp), _vp(mc), _vp(mv), k,
                                  _vp(labels), _vp(top1), _vp(top2), _vp(ctr), threads)
    if rc:
        raise RuntimeError("oracle_assign_ivf failed")
    return labels, top1, top2, int(ctr[0])


def ref_kernels():
    """The reference's own compiled Cython kernel module built into oracle/_ref
    (oracle/build_ref.sh), or None when it was not built."""
    so = sorted(REF_DIR.glob("_kernels*.so"))
    if not so:
        return None
    spec = importlib.util.spec_from_file_location("_kernels", so[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


# ---------------------------------------------------------------- numpy parts

@dataclass
class Means:
    """Mean-major CSR (means.py:24-64): 1-based terms, float64 values."""

    k: int
    dim: int
    indptr: np.ndarray
    term_ids: np.ndarray
    values: np.ndarray
    retained: np.ndarray

    @property
    def sum_terms(self) -> int:
        return int(self.term_ids.size)


def inverted(m: Means):
    """means.py:169-179: term-major postings, owners (1-based) ascending per term."""
    counts = np.diff(m.indptr)
    owners = np.repeat(np.arange(1, m.k + 1, dtype=np.int32), counts)
    order = np.argsort(m.term_ids, kind="stable")
    per_term = np.bincount(m.term_ids, minlength=m.dim + 1)[1:]
    indptr = np.zeros(m.dim + 1, dtype=np.int64)
    np.cumsum(per_term, out=indptr[1:])
    return indptr, owners[order], m.values[order]


def assign(ds, m: Means, threads=1):
    ip, own, val = inverted(m)
    return assign_ivf(ds.indptr, ds.term_ids, ds.values, ip, own, val, m.k, threads)


def sizes_of(labels, k):
    """variants.py:56-59."""
    return np.bincount(np.asarray(labels) - 1, minlength=k).astype(np.int64)


def _member_entry_order(ds, labels):
    """variants.py:240-251."""
    nnz_per_doc = np.diff(ds.indptr)
    order = np.argsort(labels, kind="stable")
    lens = nnz_per_doc[order]
    total = int(lens.sum())
    if total == 0:
        return np.empty(0, dtype=np.int64), order
    ends = np.cumsum(lens)
    seq = np.arange(total, dtype=np.int64)
    member = np.searchsorted(ends, seq, side="right")
    entry = seq - (ends[member] - lens[member]) + np.asarray(ds.indptr)[order[member]]
    return entry, order


def update(ds, labels, prev: Means) -> Means:
    """variants.py:254-307 update_means (float64; empty clusters retained)."""
    k = prev.k
    labels = np.asarray(labels, dtype=np.int32)
    sizes = sizes_of(labels, k)
    entry, _ = _member_entry_order(ds, labels)
    tsub = np.asarray(ds.term_ids)[entry]
    vsub = np.asarray(ds.values)[entry]
    ent_counts = np.bincount(labels - 1, weights=np.diff(ds.indptr), minlength=k).astype(np.int64)
    bounds = np.zeros(k + 1, dtype=np.int64)
    np.cumsum(ent_counts, out=bounds[1:])
    out_t, out_v = [], []
    counts = np.empty(k, dtype=np.int64)
    retained = np.zeros(k, dtype=bool)
    for j in range(k):
        size = int(sizes[j])
        if size == 0:
            s, e = int(prev.indptr[j]), int(prev.indptr[j + 1])
            out_t.append(prev.term_ids[s:e])
            out_v.append(prev.values[s:e])
            counts[j] = e - s
            retained[j] = True
            continue
        s, e = int(bounds[j]), int(bounds[j + 1])
        w = np.bincount(tsub[s:e] - 1, weights=vsub[s:e], minlength=ds.dim)
        w /= size
        nrm = np.sqrt(np.sum(w * w))
        nz = np.flatnonzero(w)
        out_t.append((nz + 1).astype(np.int32))
        out_v.append(w[nz] / nrm)
        counts[j] = nz.size
    indptr = np.zeros(k + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    terms = np.concatenate(out_t) if out_t else np.empty(0, np.int32)
    vals = np.concatenate(out_v) if out_v else np.empty(0, np.float64)
    return Means(k, ds.dim, indptr, terms.astype(np.int32), vals, retained)


def update_fast(ds, labels, prev: Means, chunk_bytes: int = 256 << 20) -> Means:
    """update() vectorised for large k (BASELINE configs 2-4), bit-identical
    to it (tests/test_oracle.py pins the two against each other):

    * the per-cluster ``bincount(tsub - 1, weights=vsub)`` of variants.py:290
      adds a cluster's entries of one term sequentially in entry order; one
      global bincount over the (cluster, term) keys' ranks adds the same
      subsequence in the same order, starting from the same 0.0;
    * ``w /= size`` and the nonzero test (variants.py:291,294) per key;
    * ``np.sum(w * w)`` (variants.py:292) is numpy's pairwise sum over the
      dense length-D vector: replayed on dense (clusters x D) chunks with
      ``np.sum(axis=1)``, which reduces each contiguous row with the same
      pairwise routine as the 1-D sum;
    * empty clusters keep the previous mean (variants.py:281-286)."""
    k, dim = prev.k, ds.dim
    labels = np.asarray(labels, dtype=np.int32)
    sizes = sizes_of(labels, k)
    entry, order = _member_entry_order(ds, labels)
    lens = np.diff(ds.indptr)[order]
    lab_e = np.repeat(labels[order].astype(np.int64) - 1, lens)
    tsub = np.asarray(ds.term_ids)[entry].astype(np.int64) - 1
    vsub = np.asarray(ds.values)[entry]
    keys, inv = np.unique(lab_e * dim + tsub, return_inverse=True)
    sums = np.bincount(inv.ravel(), weights=vsub, minlength=keys.size)
    kc = keys // dim
    kt = keys - kc * dim
    w = sums / sizes[kc].astype(np.float64)
    # pairwise norms over dense chunks of clusters (zeros included, as numpy)
    nrm = np.zeros(k)
    starts = np.searchsorted(kc, np.arange(k + 1))
    per = max(1, chunk_bytes // (8 * max(dim, 1)))
    live = np.flatnonzero(sizes > 0)
    for c0 in range(0, live.size, per):
        cl = live[c0:c0 + per]
        dense = np.zeros((cl.size, dim))
        for r, c in enumerate(cl):
            s, e = starts[c], starts[c + 1]
            dense[r, kt[s:e]] = w[s:e]
        nrm[cl] = np.sqrt(np.sum(dense * dense, axis=1))
    keep = w != 0.0
    counts = np.bincount(kc[keep], minlength=k).astype(np.int64)
    retained = sizes == 0
    pc = np.diff(prev.indptr)
    counts[retained] = pc[retained]
    indptr = np.zeros(k + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    terms = np.empty(int(indptr[-1]), np.int32)
    vals = np.empty(int(indptr[-1]), np.float64)
    kk = np.flatnonzero(keep)
    kcl = kc[kk]
    rank = np.arange(kk.size) - np.searchsorted(kcl, kcl)  # position within its cluster
    pos = indptr[kcl] + rank
    terms[pos] = (kt[kk] + 1).astype(np.int32)
    vals[pos] = w[kk] / nrm[kcl]
    for c in np.flatnonzero(retained):
        s, e = int(prev.indptr[c]), int(prev.indptr[c + 1])
        terms[indptr[c]:indptr[c + 1]] = prev.term_ids[s:e]
        vals[indptr[c]:indptr[c + 1]] = prev.values[s:e]
    return Means(k, dim, indptr, terms, vals, retained)


def objective(ds, labels, m: Means, dense_limit: int = 600_000_000) -> float:
    """clustering.py:105-119: each entry's product v * mu_{label}[t] (0 where
    the mean lacks t), per-object bincount in entry order, then math.fsum.
    Uses the reference's dense k x D gather when it fits (k*D <= dense_limit
    float64s), else the same products gathered from the sparse CSR."""
    n = ds.indptr.size - 1
    owners = np.repeat(np.arange(n), np.diff(ds.indptr))
    rows = (np.asarray(labels, np.int64) - 1)[owners]
    if m.k * m.dim <= dense_limit:  # literally clustering.py:115-119 (means.py:156-162)
        dense = np.zeros((m.k, m.dim), dtype=np.float64)
        dense[np.repeat(np.arange(m.k), np.diff(m.indptr)), m.term_ids - 1] = m.values
        contrib = np.asarray(ds.values) * dense[rows, np.asarray(ds.term_ids) - 1]
        sims = np.bincount(owners, weights=contrib, minlength=n)
        return math.fsum(sims.tolist())
    mkeys = np.repeat(np.arange(m.k, dtype=np.int64), np.diff(m.indptr)) * (m.dim + 1) + \
        m.term_ids.astype(np.int64)
    ekeys = rows * (m.dim + 1) + np.asarray(ds.term_ids, np.int64)
    pos = np.searchsorted(mkeys, ekeys)
    pos_c = np.minimum(pos, max(mkeys.size - 1, 0))
    hit = (mkeys.size > 0) & (mkeys[pos_c] == ekeys) if mkeys.size else np.zeros(ekeys.size, bool)
    u = np.where(hit, m.values[pos_c] if m.values.size else 0.0, 0.0)
    contrib = np.asarray(ds.values) * u
    sims = np.bincount(owners, weights=contrib, minlength=n)
    return math.fsum(sims.tolist())


def volume_ivf(ds, m: Means) -> int:
    """counters.py:71-81."""
    no = np.bincount(ds.term_ids, minlength=ds.dim + 1)[1:].astype(np.int64)
    nc = np.bincount(m.term_ids, minlength=m.dim + 1)[1:].astype(np.int64)
    return int(np.dot(no, nc))


class SplitMix64:
    """clustering.py:41-69."""

    M = 0xFFFFFFFFFFFFFFFF

    def __init__(self, seed):
        self.s = seed & self.M

    def next_u64(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & self.M
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
        return z ^ (z >> 31)

    def below(self, n):
        limit = (1 << 64) - ((1 << 64) % n)
        while True:
            r = self.next_u64()
            if r < limit:
                return r % n


def sample_without_replacement(n, k, seed):
    """clustering.py:72-79 (literal: arange + partial Fisher-Yates)."""
    rng = SplitMix64(seed)
    idx = np.arange(n, dtype=np.int64)
    for i in range(k):
        j = i + rng.below(n - i)
        idx[i], idx[j] = idx[j], idx[i]
    return idx[:k]


def init_means(ds, k, seed) -> Means:
    """clustering.py:82-102."""
    chosen = sample_without_replacement(ds.indptr.size - 1, k, seed)
    ip = np.asarray(ds.indptr)
    counts = ip[chosen + 1] - ip[chosen]
    indptr = np.zeros(k + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    terms = np.concatenate([ds.term_ids[ip[i]:ip[i + 1]] for i in chosen])
    vals = np.concatenate([ds.values[ip[i]:ip[i + 1]] for i in chosen])
    return Means(k, ds.dim, indptr, terms.astype(np.int32), vals.astype(np.float64),
                 np.zeros(k, dtype=bool))


def fnv1a64(labels) -> int:
    """variants.py:77-83 over labels as little-endian int32."""
    a = np.ascontiguousarray(labels, dtype="<i4")
    return int(clib().oracle_fnv1a64(C.c_void_p(a.ctypes.data), a.nbytes))


@dataclass
class OracleIter:
    index: int
    objective: float
    digest: int
    postings: int
    mean_terms_total: int
    labels: np.ndarray
    top1: np.ndarray
    top2: np.ndarray
    means: Means = field(repr=False)


@dataclass
class OracleRun:
    iters: list
    converged: bool
    final_means: Means
    final_labels: np.ndarray


def run_ivf(ds, k, seed, max_iter=50, epsilon=None, threads=1, means=None,
            variant="IVF") -> OracleRun:
    """clustering.py:229-315 for variant IVF (records hold the means that
    produced each assignment; convergence is tested before the update).
    variant="IVFD": the same similarities (IVFD adds the products in the
    same ascending term order), labels by _kernels.pyx:178-207 — the argmax
    only when it beats 0.0 (rho_max starts at 0.0), else mean 1."""
    m = means if means is not None else init_means(ds, k, seed)
    iters = []
    prev = None
    prev_obj = None
    converged = False
    for r in range(1, max_iter + 1):
        labels, top1, top2, post = assign(ds, m, threads)
        if variant == "IVFD":
            labels = np.where(top1 > 0.0, labels, 1).astype(np.int32)
        obj = objective(ds, labels, m)
        iters.append(OracleIter(r, obj, fnv1a64(labels), post, m.sum_terms, labels, top1, top2, m))
        if prev is not None and np.array_equal(labels, prev):
            converged = True
            break
        if epsilon is not None and prev_obj is not None and obj - prev_obj <= epsilon:
            converged = True
            break
        new_m = update(ds, labels, m)
        prev, prev_obj, m = labels, obj, new_m
    return OracleRun(iters, converged, m, iters[-1].labels)
