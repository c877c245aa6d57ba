"""Ingestion before the Lloyd path: UCI bag-of-words -> tf-idf unit vectors.

Mirrors reference io.py (``ParseError``, ``RawCounts``, ``parse_uci_bow``,
``tfidf_normalize``; io.py:26-174) with the work moved to native code:

* parsing runs in C++ over the whole buffer on all host threads
  (``ivfkm_uci_parse``, csrc/ingest.cpp); errors come back as (line, code,
  values) and are raised here with the reference's wording and line numbers;
* the triple sort, the duplicate-pair check, document frequencies and the
  tf-idf weighting + L2 normalisation run on the GPU (csrc/ingest.cu),
  bit-identical to the reference's numpy (the D idf logarithms are taken
  with numpy on the host exactly as io.py:141-142 does, so ``np.log``'s
  rounding is the reference's own).

``RawCounts`` keeps the triples as three sorted arrays; ``.triples`` builds
the reference's tuple-of-tuples form on demand (small inputs).
"""

from __future__ import annotations

import ctypes as C
import os
import warnings
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _lib
from .types import Dataset

__all__ = ["ParseError", "RawCounts", "parse_uci_bow", "tfidf_normalize", "load_uci_bow"]


class ParseError(ValueError):
    """Malformed input; ``line`` is the 1-based offending line number (io.py:26-33)."""

    def __init__(self, message: str, line: int | None = None):
        self.line = line
        if line is not None:
            message = f"line {line}: {message}"
        super().__init__(message)


@dataclass(frozen=True, eq=False)
class RawCounts:
    """Parsed bag-of-words triples sorted by (doc, term) (io.py:36-42)."""

    n_docs: int
    dim: int
    docs: np.ndarray    # int64, 1-based
    terms: np.ndarray   # int32, 1-based
    counts: np.ndarray  # int64
    _device: object = field(default=None, repr=False, compare=False)

    @property
    def triples(self) -> tuple:
        return tuple(zip(self.docs.tolist(), self.terms.tolist(), self.counts.tolist()))


def _read_bytes(source) -> bytes:
    """io.py:45-50: a str/Path names a file; otherwise a text stream or an
    iterable of lines."""
    if isinstance(source, (str, Path)):
        return Path(source).read_bytes()
    if hasattr(source, "read"):
        data = source.read()
        return data.encode("utf-8") if isinstance(data, str) else bytes(data)
    return "".join(source).encode("utf-8")


def _line_text(data: bytes, line: int) -> str:
    """The 1-based line, stripped, as the reference would print it."""
    start = 0
    for _ in range(line - 1):
        nl = data.find(b"\n", start)
        if nl < 0:
            return ""
        start = nl + 1
    nl = data.find(b"\n", start)
    raw = data[start:] if nl < 0 else data[start:nl]
    return raw.decode("utf-8", errors="replace").strip()


def _device():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("ingestion needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _p(t):
    return C.c_void_p(t.data_ptr())


@dataclass
class _HostParse:
    data: bytes
    header: np.ndarray
    docs: np.ndarray
    terms: np.ndarray
    counts: np.ndarray
    lines: np.ndarray
    n_read: int
    n_lines: int
    err_line: int
    err_code: int
    err_val: np.ndarray


def _parse_host(data: bytes, threads: int = 0) -> _HostParse:
    """The host half of parse_uci_bow: every check but the duplicate pairs."""
    lib = _lib.load()
    cap = data.count(b"\n") + 1
    header = np.zeros(3, np.int64)
    docs = np.empty(cap, np.int32)
    terms = np.empty(cap, np.int32)
    counts = np.empty(cap, np.int32)
    lines = np.empty(cap, np.int64)
    n_read, n_lines, err_line = C.c_int64(0), C.c_int64(0), C.c_int64(0)
    err_code = C.c_int(0)
    err_val = np.zeros(3, np.int64)
    buf = C.create_string_buffer(data, len(data))
    rc = lib.ivfkm_uci_parse(buf, len(data), threads, header.ctypes.data, cap,
                             docs.ctypes.data, terms.ctypes.data, counts.ctypes.data,
                             lines.ctypes.data, C.byref(n_read), C.byref(n_lines),
                             C.byref(err_line), C.byref(err_code), err_val.ctypes.data)
    _lib.check(rc, "ivfkm_uci_parse")
    return _HostParse(data, header, docs, terms, counts, lines, n_read.value, n_lines.value,
                      err_line.value, err_code.value, err_val)


def _raise_header(hp: _HostParse) -> None:
    if hp.err_code == 1:
        raise ParseError(f"expected a single integer, got {_line_text(hp.data, hp.err_line)!r}",
                         hp.err_line)
    if hp.err_code == 2:
        raise ParseError("header counts must be nonnegative", hp.err_line)
    if hp.n_lines == 0:
        raise ParseError("empty input", 1)
    if hp.n_lines < 3:
        raise ParseError("truncated header", hp.n_lines + 1)


def _raise_body(hp: _HostParse) -> None:
    """A malformed line (codes 3-7), else an entry-count mismatch."""
    code, eline = hp.err_code, hp.err_line
    n_docs, dim, nnz = (int(x) for x in hp.header)
    if code:
        d, t, cnt = (int(x) for x in hp.err_val)
        msg = {3: lambda: f"expected 'doc term count', got {_line_text(hp.data, eline)!r}",
               4: lambda: f"non-integer field in {_line_text(hp.data, eline)!r}",
               5: lambda: f"doc id {d} outside 1..{n_docs}",
               6: lambda: f"term id {t} outside 1..{dim}",
               7: lambda: f"count must be positive, got {cnt}"}[code]()
        raise ParseError(msg, eline)
    if hp.n_read != nnz:
        raise ParseError(f"header declares {nnz} entries but {hp.n_read} were read", hp.n_lines)


def parse_uci_bow(source, threads: int = 0) -> RawCounts:
    """Parse a UCI bag-of-words input into sorted, validated triples
    (io.py:72-121): same checks, same error messages and line numbers."""
    import torch

    lib = _lib.load()
    hp = _parse_host(_read_bytes(source), threads)
    _raise_header(hp)
    header, docs, terms, counts, lines = hp.header, hp.docs, hp.terms, hp.counts, hp.lines
    eline = hp.err_line
    n_docs, dim, nnz = (int(x) for x in header)
    n = hp.n_read
    # device: sort by (doc, term) (stable over line order) + duplicate check
    dev = _device()
    d_docs = torch.from_numpy(docs[:n]).to(dev)
    d_terms = torch.from_numpy(terms[:n]).to(dev)
    d_counts = torch.from_numpy(counts[:n]).to(dev)
    d_lines = torch.from_numpy(lines[:n]).to(dev)
    dup = torch.empty(1, dtype=torch.int64, device=dev)
    ws = torch.empty(int(lib.ivfkm_bow_workspace_size(n)), dtype=torch.uint8, device=dev)
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(lib.ivfkm_bow_sort(n, n_docs, dim, _p(d_docs), _p(d_terms), _p(d_counts),
                                  _p(d_lines), _p(dup), _p(ws), ws.numel(), stream),
               "ivfkm_bow_sort")
    dup_line = int(dup.item())  # UINT64_MAX (read as -1): no repeated pair
    has_dup = dup_line >= 0
    if has_dup and (eline < 0 or dup_line < eline):
        at = int(torch.nonzero(d_lines == dup_line)[0].item())
        raise ParseError(f"duplicate (doc, term) pair ({int(d_docs[at])}, {int(d_terms[at])})",
                         dup_line)
    _raise_body(hp)
    raw = RawCounts(n_docs, dim, d_docs.cpu().numpy().astype(np.int64),
                    d_terms.cpu().numpy().copy(), d_counts.cpu().numpy().astype(np.int64),
                    _device=(d_docs, d_terms, d_counts))
    return raw


def tfidf_normalize(raw: RawCounts) -> Dataset:
    """Weight raw counts by tf-idf and project onto the unit hypersphere
    (io.py:124-174): idf = ln(n_docs / df); zero-weight entries and the
    documents they empty are dropped (with the reference's warning)."""
    import torch

    if raw.n_docs < 1:
        if raw.docs.size:
            raise ValueError("triples present but document count is zero")
        return Dataset(raw.dim, np.zeros(1, np.int64), np.zeros(0, np.int32),
                       np.zeros(0, np.float64), normalized=True)
    lib = _lib.load()
    dev = _device()
    if raw._device is not None:
        d_docs, d_terms, d_counts = raw._device
    else:
        d_docs = torch.from_numpy(np.ascontiguousarray(raw.docs, np.int32)).to(dev)
        d_terms = torch.from_numpy(np.ascontiguousarray(raw.terms, np.int32)).to(dev)
        d_counts = torch.from_numpy(np.ascontiguousarray(np.minimum(raw.counts, 2**31 - 1),
                                                         np.int32)).to(dev)
    n, n_docs, dim = int(d_docs.numel()), raw.n_docs, raw.dim
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    df = torch.empty(max(dim, 1), dtype=torch.int64, device=dev)
    _lib.check(lib.ivfkm_bow_df(n, dim, _p(d_terms), _p(df), stream), "ivfkm_bow_df")
    dfh = df.cpu().numpy()[:dim]
    # io.py:141-142, the reference's own arithmetic (D logarithms)
    idf = np.zeros(dim, dtype=np.float64)
    nz = dfh > 0
    idf[nz] = np.log(n_docs / dfh[nz])
    d_idf = torch.from_numpy(idf if dim else np.zeros(1)).to(dev)
    out_ptr = torch.empty(n_docs + 1, dtype=torch.int64, device=dev)
    out_terms = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    out_vals = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    dropped = torch.empty(max(n_docs, 1), dtype=torch.int32, device=dev)
    cnt = np.zeros(2, np.int64)
    ws = torch.empty(int(lib.ivfkm_tfidf_workspace_size(n, n_docs)), dtype=torch.uint8,
                     device=dev)
    _lib.check(lib.ivfkm_tfidf(n, n_docs, dim, _p(d_docs), _p(d_terms), _p(d_counts), _p(d_idf),
                               _p(out_ptr), _p(out_terms), _p(out_vals), _p(dropped),
                               cnt.ctypes.data, _p(ws), ws.numel(), stream), "ivfkm_tfidf")
    n_alive, kept = int(cnt[0]), int(cnt[1])
    drop = tuple(int(x) for x in dropped[: n_docs - n_alive].cpu().numpy())
    if drop:
        warnings.warn(f"dropped {len(drop)} document(s) with no nonzero tf-idf weight",
                      stacklevel=2)
    return Dataset(dim, out_ptr[: n_alive + 1].cpu().numpy(), out_terms[:kept].cpu().numpy(),
                   out_vals[:kept].cpu().numpy(), normalized=True, dropped_docs=drop)


def load_uci_bow(path: str | os.PathLike, threads: int = 0) -> Dataset:
    """parse_uci_bow + tfidf_normalize (the reference CLI's ``ingest`` step)."""
    return tfidf_normalize(parse_uci_bow(Path(path), threads=threads))
