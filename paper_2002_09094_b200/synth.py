"""Seeded synthetic corpora shaped like BASELINE.json's five configs.

PubMed / NYT (the paper's corpora) are not available
offline, so every benchmark and parity case runs on a seeded stand-in whose
shapes and value distributions follow BASELINE.json:configs (restated in
SURVEY.md §8(d)).  Generation is native (csrc/synth.cpp, OpenMP; every row
has its own SplitMix64 stream, so the output does not depend on the thread
count):

* per-row nnz: Poisson(mean) or lognormal(distribution mean, sigma), clipped;
* term ids: first nnz_i distinct draws of a Zipf(s) sequence over 1..D
  (successive sampling without replacement), sorted;
* values: tf-idf ``(1 + ln count) * ln(N / df)``, ``count ~ Geometric(1/2)``;
  df == N terms (weight 0) are dropped as the reference ingestion does
  (io.py:153-154), rows left empty are dropped (io.py:156-164);
* rows L2-normalised in float64 (the reference checks 1e-12, data.py:165-172).

Output follows the reference conventions: int64 indptr, 1-based int32 term
ids strictly increasing per row, float64 values.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["CorpusSpec", "CONFIGS", "make_corpus", "make_dataset", "config_spec"]


@dataclass(frozen=True)
class CorpusSpec:
    n: int
    dim: int
    nnz_kind: str          # "poisson" | "lognormal"
    nnz_mean: float
    nnz_sigma: float       # lognormal only
    nnz_lo: int
    nnz_hi: int
    zipf_s: float
    seed: int

    def scaled(self, n: int, dim: int | None = None, seed: int | None = None) -> "CorpusSpec":
        """Same distributions on a smaller shape (parity tests)."""
        return CorpusSpec(n, dim or self.dim, self.nnz_kind, self.nnz_mean, self.nnz_sigma,
                          self.nnz_lo, self.nnz_hi, self.zipf_s,
                          self.seed if seed is None else seed)


# Data shapes; configs 1/2 and 3/4 share their corpus (BASELINE.json:configs).
_C0 = CorpusSpec(20_000, 10_000, "poisson", 40.0, 0.0, 1, 200, 1.1, 1000)
_C12 = CorpusSpec(300_000, 100_000, "lognormal", 230.0, 0.6, 5, 2000, 1.1, 1001)
_C34 = CorpusSpec(8_200_000, 141_000, "poisson", 59.0, 0.0, 1, 1000, 1.05, 1003)

#: config index -> corpus, k, iterations, mean seed
CONFIGS = {
    0: dict(corpus=_C0, k=100, iters=10, seed=1),
    1: dict(corpus=_C12, k=1_000, iters=50, seed=1),
    2: dict(corpus=_C12, k=10_000, iters=20, seed=1),
    3: dict(corpus=_C34, k=10_000, iters=10, seed=1),
    4: dict(corpus=_C34, k=60_000, iters=5, seed=1),
}


def config_spec(index: int) -> dict:
    return CONFIGS[index]


_corpus = None


def corpus_lib():
    """The generator alone (tools/_build/libcorpus.so: csrc/synth.cpp without
    CUDA) — for processes that must not map libivfkm.so (bench.py's
    reference arm).  Same code, same output."""
    global _corpus
    if _corpus is None:
        from .build import CORPUS_LIB, build_corpus_library

        if not CORPUS_LIB.exists():
            build_corpus_library()
        lib = C.CDLL(str(CORPUS_LIB))
        for name in ("ivfkm_synth_rows", "ivfkm_synth_fill"):
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = _lib.SIGNATURES[name]
        _corpus = lib
    return _corpus


def make_corpus(spec: CorpusSpec, standalone: bool = False):
    """(indptr int64[N+1], term_ids int32 1-based, values float64, n dropped rows).

    ``standalone``: generate with corpus_lib() instead of libivfkm.so."""
    lib = corpus_lib() if standalone else _lib.load()
    cs = _lib.SynthSpec(spec.n, spec.dim, 0 if spec.nnz_kind == "poisson" else 1,
                        spec.nnz_mean, spec.nnz_sigma, spec.nnz_lo, spec.nnz_hi, spec.zipf_s,
                        spec.seed)
    rows = np.empty(spec.n, dtype=np.int64)
    _lib.check(lib.ivfkm_synth_rows(C.byref(cs), C.c_void_p(rows.ctypes.data)), "synth_rows")
    cap = np.zeros(spec.n + 1, dtype=np.int64)
    np.cumsum(rows, out=cap[1:])
    total = int(cap[-1])
    indptr = np.empty(spec.n + 1, dtype=np.int64)
    terms = np.empty(total, dtype=np.int32)
    vals = np.empty(total, dtype=np.float64)
    n_out, nnz_out = C.c_int64(0), C.c_int64(0)
    _lib.check(lib.ivfkm_synth_fill(C.byref(cs), C.c_void_p(cap.ctypes.data),
                                    C.c_void_p(indptr.ctypes.data), C.c_void_p(terms.ctypes.data),
                                    C.c_void_p(vals.ctypes.data), C.byref(n_out),
                                    C.byref(nnz_out)), "synth_fill")
    n, nnz = n_out.value, nnz_out.value
    return indptr[: n + 1].copy(), terms[:nnz].copy(), vals[:nnz].copy(), spec.n - n


def make_dataset(spec: CorpusSpec, dataset_cls=None, standalone: bool = False):
    """Generate a corpus and wrap it in a (reference-compatible) Dataset."""
    if dataset_cls is None:
        from .types import Dataset as dataset_cls  # noqa: N813
    indptr, terms, vals, _ = make_corpus(spec, standalone)
    return dataset_cls(spec.dim, indptr, terms, vals, normalized=True)
