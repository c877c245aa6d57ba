"""Device-resident Lloyd engine: objects, means and every per-iteration
buffer live in HBM; the host only launches the C-ABI kernels and reads a
few bytes of statistics per iteration.

One Lloyd iteration (the reference's loop body, clustering.py:262-298):

    assign   ivfkm_assign        fp32 register screen + exact fp64 rescoring,
                                 changed-label count, sizes, exact objective
    (host)   read ivfkm_stats    convergence decision, objective, V
    update   ivfkm_update_count  sort/segment-sum/normalise (bit-exact)
             ivfkm_update_fill   new mean-major CSR (+ retained copies)
             ivfkm_bivf_build    new bitmap-block inverted file

torch is used for device memory, pinned host buffers and the current CUDA
stream only; all compute on the path is in libivfkm.so.
"""

from __future__ import annotations

import ctypes as C
import os
import warnings
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .types import MeanSet

__all__ = ["DeviceDataset", "DeviceMeans", "LloydEngine", "IterStats", "objective_from_limbs"]

_MU_MAX = 1.0 + 1e-9  # means are unit norm to 1e-12 (means.py:56-60)


def _p(t: torch.Tensor | None) -> C.c_void_p | None:
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream() -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def objective_from_limbs(limbs) -> float:
    """Round the exact fixed-point sum (limb l weighs 2^(32 l - 1074)) once to
    the nearest double: the same value math.fsum returns (clustering.py:119)."""
    x = 0
    for i, v in enumerate(limbs):
        x += int(v) << (32 * i)
    return x / (1 << 1074)  # int/int true division is correctly rounded


@dataclass
class IterStats:
    postings: int
    changed: int
    near_ties: int
    overflow: int
    objective: float

    @classmethod
    def from_raw(cls, s: "_lib.Stats") -> "IterStats":
        if s.obj_flags:
            raise FloatingPointError("objective summand outside the exact accumulator range")
        return cls(int(s.postings), int(s.changed), int(s.near_ties), int(s.overflow),
                   objective_from_limbs(s.obj_limbs))


def encode_row_gaps(ip: np.ndarray, terms0: np.ndarray):
    """Sorted 0-based row terms as 16-bit gaps (ivfkm_rows_decode's format):
    (gaps uint16[nnz], exception positions int64, their absolute ids int32)."""
    g = np.empty(terms0.size, np.int64)
    if terms0.size:
        g[1:] = np.diff(terms0.astype(np.int64))
        starts = ip[:-1][np.diff(ip) > 0]
        g[starts] = terms0[starts].astype(np.int64) + 1
    exc = np.flatnonzero(g >= 0xFFFF)
    gaps = np.where(g >= 0xFFFF, 0xFFFF, g).astype(np.uint16)
    return gaps, exc.astype(np.int64), terms0[exc].astype(np.int32)


class HostDataset:
    """Pinned host copies of the device layout (for end-to-end transfers).

    ``compact``: keep the term ids as 16-bit in-row gaps (+ a short exception
    list) instead of int32 — the device decodes them (ivfkm_rows_decode), so
    a step's corpus upload moves 2 bytes per term instead of 4."""

    def __init__(self, ds, pin: bool = True, compact: bool = False):
        ip = np.ascontiguousarray(ds.indptr, dtype=np.int64)
        self.n = int(ip.size - 1)
        self.dim = int(ds.dim)
        self.nnz = int(ip[-1])
        terms0 = np.ascontiguousarray(ds.term_ids, dtype=np.int32) - 1
        vals = np.ascontiguousarray(ds.values, dtype=np.float64)
        rows = np.diff(ip)
        xn = np.sqrt(np.bincount(np.repeat(np.arange(self.n), rows), weights=vals * vals,
                                 minlength=self.n)) if self.n else np.zeros(0)
        self.max_row = int(rows.max()) if self.n else 0

        def host(a):
            t = torch.from_numpy(np.array(a, copy=True))
            return t.pin_memory() if pin else t

        self.row_ptr = host(ip)
        self.compact = bool(compact)
        if self.compact:
            gaps, exc_idx, exc_term = encode_row_gaps(ip, terms0)
            self.gaps = host(gaps.view(np.int16))
            self.exc_idx = host(exc_idx if exc_idx.size else np.zeros(1, np.int64))
            self.exc_term = host(exc_term if exc_term.size else np.zeros(1, np.int32))
            self.n_exc = int(exc_idx.size)
            self.terms = None
        else:
            self.terms = host(terms0.astype(np.int32))
        self.val64 = host(vals)
        self.xnorm = host(xn.astype(np.float64))

    def _arrays(self):
        if self.compact:
            return (self.row_ptr, self.gaps, self.exc_idx, self.exc_term, self.val64, self.xnorm)
        return (self.row_ptr, self.terms, self.val64, self.xnorm)

    @property
    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self._arrays())


# host threads that fill / drain the pinned staging buffers (one thread's
# memcpy runs at a fraction of the PCIe bandwidth); numpy copies release the GIL
UPLOAD_THREADS = max(1, min(8, os.cpu_count() or 1))
_POOL: ThreadPoolExecutor | None = None


def _pcopy(dst: np.ndarray, src: np.ndarray) -> None:
    """dst[:] = src over UPLOAD_THREADS host threads (1-D byte views)."""
    global _POOL
    n, th = dst.size, UPLOAD_THREADS
    if th <= 1 or n < (4 << 20):
        dst[:] = src
        return
    if _POOL is None or _POOL._max_workers < th:
        _POOL = ThreadPoolExecutor(max(th, 8))
    step = -(-n // th)
    futs = [_POOL.submit(np.copyto, dst[i:i + step], src[i:i + step]) for i in range(0, n, step)]
    for f in futs:
        f.result()


def _upload(a: np.ndarray, dev, chunk: int = 64 << 20) -> torch.Tensor:
    """Host array -> device through two pinned staging buffers (chunked,
    asynchronous, double-buffered, each stage filled by several host
    threads): pageable copies run at a fraction of the PCIe bandwidth."""
    a = np.ascontiguousarray(a)
    with warnings.catch_warnings():  # read-only reference arrays: only read here
        warnings.simplefilter("ignore", UserWarning)
        out = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, device=dev)
    nbytes = a.nbytes
    if nbytes <= chunk or not torch.cuda.is_available():
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", UserWarning)
            out.copy_(torch.from_numpy(a))
        return out
    src = a.reshape(-1).view(np.uint8)
    dst = out.view(-1).view(torch.uint8)
    stage = [torch.empty(chunk, dtype=torch.uint8).pin_memory() for _ in range(2)]
    done = [None, None]
    st = torch.cuda.current_stream()
    for i, off in enumerate(range(0, nbytes, chunk)):
        b = i & 1
        if done[b] is not None:
            done[b].synchronize()  # the copy out of this staging buffer has finished
        n = min(chunk, nbytes - off)
        _pcopy(stage[b][:n].numpy(), src[off:off + n])
        dst[off:off + n].copy_(stage[b][:n], non_blocking=True)
        done[b] = torch.cuda.Event()
        done[b].record(st)
    st.synchronize()
    return out


def _download(t: torch.Tensor, chunk: int = 64 << 20) -> np.ndarray:
    """Device tensor -> new host array through two pinned staging buffers:
    the copy of chunk i+1 runs while host threads drain chunk i."""
    t = t.contiguous().reshape(-1)
    if t.numel() * t.element_size() <= chunk or not t.is_cuda:
        return t.cpu().numpy()
    out = np.empty(t.numel(), dtype=torch.empty(0, dtype=t.dtype).numpy().dtype)
    nbytes = out.nbytes
    src = t.view(torch.uint8)
    dst = out.view(np.uint8)
    stage = [torch.empty(chunk, dtype=torch.uint8).pin_memory() for _ in range(2)]
    st = torch.cuda.current_stream()
    pending = []
    for i, off in enumerate(range(0, nbytes + chunk, chunk)):
        if off < nbytes:
            n = min(chunk, nbytes - off)
            stage[i & 1][:n].copy_(src[off:off + n], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(st)
            pending.append((i & 1, off, n, ev))
        if pending and (len(pending) == 2 or off >= nbytes):
            b, o, n, ev = pending.pop(0)
            ev.synchronize()
            _pcopy(dst[o:o + n], stage[b][:n].numpy())
    return out


class DeviceDataset:
    """Objects on the device: int64 row_ptr, 0-based int32 terms, fp32 values
    (screening) and fp64 values (rescoring, update), fp64 row norms."""

    def __init__(self, host: HostDataset, device: torch.device | str = "cuda",
                 copies_only: bool = False):
        """``copies_only``: issue the host->device copies and stop; finish()
        runs the kernels (term decode, fp32 cast) later, e.g. on the compute
        stream — on a copy stream a kernel waits for free SMs behind the
        compute kernels and delays the step that needs it."""
        self.n, self.dim, self.nnz, self.max_row = host.n, host.dim, host.nnz, host.max_row
        self.device = torch.device(device)
        nb = host.row_ptr.is_pinned()
        # every host->device copy first, then the kernels (decode, fp32 cast):
        # on a copy stream a kernel waits for free SMs, and a copy queued
        # behind it would wait with it
        self.row_ptr = host.row_ptr.to(self.device, non_blocking=nb)
        if host.compact:
            gaps = host.gaps.to(self.device, non_blocking=nb)
            exc_idx = host.exc_idx.to(self.device, non_blocking=nb)
            exc_term = host.exc_term.to(self.device, non_blocking=nb)
        else:
            self.terms = host.terms.to(self.device, non_blocking=nb)
        self.val64 = host.val64.to(self.device, non_blocking=nb)
        self.xnorm = host.xnorm.to(self.device, non_blocking=nb)
        self._pending = (gaps, exc_idx, exc_term, host.n_exc) if host.compact else ()
        self.val32 = None
        if not copies_only:
            self.finish()

    def finish(self) -> "DeviceDataset":
        """Kernels after the copies, on the current stream: decode the
        compact term ids (ivfkm_rows_decode), cast the fp32 screen values."""
        if self._pending:
            gaps, exc_idx, exc_term, n_exc = self._pending
            terms = torch.empty(max(self.nnz, 1), dtype=torch.int32, device=self.device)
            _lib.check(_lib.load().ivfkm_rows_decode(
                self.n, _p(self.row_ptr), _p(gaps), n_exc, _p(exc_idx), _p(exc_term), _p(terms),
                _stream()), "ivfkm_rows_decode")
            for t in (gaps, exc_idx, exc_term):  # allocated on the copying stream
                t.record_stream(torch.cuda.current_stream())
            self.terms = terms[:self.nnz]
            self._pending = ()
        if self.val32 is None:
            self.val32 = self.val64.to(torch.float32)
        return self

    @classmethod
    def from_dataset(cls, ds, device="cuda") -> "DeviceDataset":
        """Upload a reference Dataset's own arrays (no host-side conversion) and
        derive the device layout there (ivfkm_rows_prepare)."""
        self = cls.__new__(cls)
        dev = torch.device(device)
        ip = np.ascontiguousarray(ds.indptr, dtype=np.int64)
        t1 = np.ascontiguousarray(ds.term_ids, dtype=np.int32)
        v = np.ascontiguousarray(ds.values, dtype=np.float64)
        self.n, self.dim, self.nnz = int(ip.size - 1), int(ds.dim), int(ip[-1])
        self.max_row = int(np.diff(ip).max()) if self.n else 0
        self.device = dev
        self.row_ptr = _upload(ip, dev)
        self.terms = _upload(t1, dev)  # 1-based; made 0-based in place below
        self.val64 = _upload(v, dev)
        self.val32 = torch.empty(max(self.nnz, 1), dtype=torch.float32, device=dev)[:self.nnz]
        self.xnorm = torch.empty(max(self.n, 1), dtype=torch.float64, device=dev)[:self.n]
        self._pending = ()
        _lib.check(_lib.load().ivfkm_rows_prepare(
            self.n, _p(self.row_ptr), _p(self.terms), _p(self.val64), _p(self.terms),
            _p(self.val32), _p(self.xnorm), _stream()), "ivfkm_rows_prepare")
        return self


class DeviceMeans:
    """Means on the device: mean-major CSR (fp64, 0-based terms) + BIVF."""

    def __init__(self, k, dim, ptr, terms, vals, retained):
        self.k, self.dim = int(k), int(dim)
        self.ptr, self.terms, self.vals, self.retained = ptr, terms, vals, retained
        self.nnz = int(terms.numel())
        self.headers = self.pvs = self.pv64 = None
        self.slot8 = None  # sparse spans' slot bytes (ivfkm_bivf_slots), or None
        self.dir_ready = None  # event: the engine's rank directory holds these means'
        self.screen_bits = 32  # precision of pvs (the screen's values), set by build_bivf

    @classmethod
    def from_meanset(cls, ms, device="cuda") -> "DeviceMeans":
        dev = torch.device(device)
        ptr = torch.from_numpy(np.array(ms.indptr, dtype=np.int64)).to(dev)
        terms = torch.from_numpy(np.array(ms.term_ids, dtype=np.int32) - 1).to(dev)
        vals = torch.from_numpy(np.array(ms.values, dtype=np.float64)).to(dev)
        ret = torch.from_numpy(np.array(ms.retained, dtype=np.uint8)).to(dev)
        return cls(ms.k, ms.dim, ptr, terms, vals, ret)

    def to_meanset(self, representation: str = "sparse_inverted", validate: bool = True) -> MeanSet:
        ptr = self.ptr.cpu().numpy()
        terms = _download(self.terms)
        terms += 1
        vals = _download(self.vals)
        ret = self.retained.cpu().numpy().astype(bool)
        if not validate:
            return MeanSet.trusted(self.k, self.dim, representation, ptr, terms, vals, ret)
        return MeanSet(self.k, self.dim, representation, ptr, terms, vals, ret)


# kernels every update launches after its sort: the run scan (init + sweep),
# run sums (+ the cluster and leaf-group run tables), long runs, the nonzero
# scan (2), norm, the counts scan (2), fill, retain
_UPDATE_COMMON = 11


def update_launches(k: int, dim: int) -> int:
    """Kernels one stateless update launches: keys, CUB onesweep radix sort
    (histogram, exclusive sum, one pass per 8 key bits), then the common
    kernels."""
    bits = max(1, int(np.ceil(np.log2(max(2.0, float(k) * float(dim))))))
    return 3 + (bits + 7) // 8 + _UPDATE_COMMON


def delta_update_launches(k: int, dim: int) -> int:
    """Kernels of an update through the label-delta sort when few objects
    moved: changed flags, the movers' list (CUB select: 2), their lengths and
    offsets (scan: 2), their keys, their radix sort over the (label, term)
    bits (histogram, exclusive sum, a pass per 8 bits), the merge with
    deletions (tile searches, tile counts, their scan (2), merge), header;
    then the common kernels."""
    bits = int(np.ceil(np.log2(max(2, k)))) + int(np.ceil(np.log2(max(2, dim))))
    return 15 + (bits + 7) // 8 + _UPDATE_COMMON


def update_rows(lib, n_obj, nnz, row_ptr, terms, val64, labels0, sizes, prev: DeviceMeans, k,
                dim, ws, total_host=None, state=None, deferred=False) -> DeviceMeans:
    """Bit-exact update (variants.py:254-307) of k means from n_obj device rows
    whose 0-based labels lie in [0, k): ivfkm_update_count (or, with a
    label-delta ``state``, ivfkm_update_count_delta), one 8-byte device->host
    read of the new size, ivfkm_update_fill.  No BIVF.

    ``deferred``: skip the size read; the mean arrays get a capacity bound
    (new nonzeros <= runs <= nnz, plus retained means' previous postings) and
    ``nnz`` stays -1 until build_bivf, whose plan returns the exact count."""
    dev = row_ptr.device
    new_ptr = torch.empty(k + 1, dtype=torch.int64, device=dev)
    if state is not None:
        rc = lib.ivfkm_update_count_delta(n_obj, nnz, _p(row_ptr), _p(terms), _p(val64), k, dim,
                                          _p(labels0), _p(sizes), _p(prev.ptr), _p(new_ptr),
                                          _p(ws), ws.numel(), _p(state), state.numel(),
                                          _stream())
        _lib.check(rc, "ivfkm_update_count_delta")
    else:
        rc = lib.ivfkm_update_count(n_obj, nnz, _p(row_ptr), _p(terms), _p(val64), k, dim,
                                    _p(labels0), _p(sizes), _p(prev.ptr), _p(new_ptr), _p(ws),
                                    ws.numel(), _stream())
        _lib.check(rc, "ivfkm_update_count")
    if deferred:
        total = min(nnz + prev.nnz, k * dim)
    else:
        if total_host is None:
            total_host = torch.zeros(1, dtype=torch.int64)
        total_host.copy_(new_ptr[k:], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        total = int(total_host[0])
    t = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    v = torch.empty(max(total, 1), dtype=torch.float64, device=dev)
    ret = torch.empty(k, dtype=torch.uint8, device=dev)
    rc = lib.ivfkm_update_fill(n_obj, nnz, k, dim, _p(sizes), _p(prev.ptr), _p(prev.terms),
                               _p(prev.vals), _p(new_ptr), _p(t), _p(v), _p(ret), total, _p(ws),
                               ws.numel(), _stream())
    _lib.check(rc, "ivfkm_update_fill")
    out = DeviceMeans(k, dim, new_ptr, t[:total], v[:total], ret)
    if deferred:
        out.nnz = -1
    return out


class LloydEngine:
    """Runs IVF Lloyd iterations over one device-resident dataset."""

    def __init__(self, dd: DeviceDataset, k: int, screen_bits: int = 16,
                 delta_update: bool = True, update_ws: bool = True):
        self.lib = _lib.load()
        self.dd, self.k = dd, int(k)
        # fp16 screen values: half the posting bytes, a wider (still rigorous)
        # error window, labels unchanged; 32 = fp32 screen
        self.screen_bits = screen_bits
        dev = dd.device
        self.device = dev
        n, nnz, dim = dd.n, dd.nnz, dd.dim
        self.nblk = int(self.lib.ivfkm_bivf_nblk(self.k))
        u8 = torch.uint8
        self.ws_assign = torch.empty(int(self.lib.ivfkm_assign_workspace_size(n, self.k)),
                                     dtype=u8, device=dev)
        # update_ws=False: a caller that updates other rows (dist.py) brings its own
        self.ws_update = torch.empty(int(self.lib.ivfkm_update_workspace_size(n, nnz, self.k,
                                                                              dim)),
                                     dtype=u8, device=dev) if update_ws else None
        self.ws_bivf = torch.empty(int(self.lib.ivfkm_bivf_workspace_size(dim, self.k)),
                                   dtype=u8, device=dev)
        self.ws_fill = None  # sorted BIVF fill (grows with the means' size)
        # rank directory of the means' CSR for the exact rescoring (one lookup
        # word per 32 terms per mean): config 1 +1%, config 2 +0.6%; not at
        # config 4's 2 GB
        nw = (dim + 31) // 32
        self.rankdir = (torch.empty(self.k * nw * 2, dtype=torch.int32, device=dev)
                        if self.k * nw * 8 <= (512 << 20) else None)
        # the directory depends on the means only: it is built on a side
        # stream as soon as the means exist, under the BIVF build and the screen
        self.side = torch.cuda.Stream(device=dev) if self.rankdir is not None and \
            torch.cuda.is_available() else None
        self._dir_of = None  # the means whose directory the buffer holds (side-stream build)
        # BIVF value arrays, grown on demand and alternated between builds (the
        # means of the previous build keep theirs)
        self._bvbuf = [None, None]
        self._bvpar = 0
        self._totals = np.zeros(2, np.int64)
        # label-delta update sort: the previous iteration's sorted entries
        # (DESIGN.md §4); zero-filled = no state yet
        sbytes = int(self.lib.ivfkm_update_state_size(n, nnz, self.k, dim)) if delta_update else 0
        self.upd_state = torch.zeros(sbytes, dtype=u8, device=dev) if sbytes else None
        self.labels = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(2)]
        self.cur = 0
        self.sims = torch.empty(n, dtype=torch.float64, device=dev)
        self.sizes = torch.empty(self.k, dtype=torch.int64, device=dev)  # unsigned on device
        self.stats = torch.zeros(C.sizeof(_lib.Stats), dtype=u8, device=dev)
        self.stats_host = torch.zeros(C.sizeof(_lib.Stats), dtype=u8).pin_memory() \
            if torch.cuda.is_available() else torch.zeros(C.sizeof(_lib.Stats), dtype=u8)
        self.total_host = torch.zeros(1, dtype=torch.int64).pin_memory()
        self.rowcap = max(32, min(512, (dd.max_row + 31) // 32 * 32))
        self.order = self._row_order(dd)
        self.launches = 0  # our kernels launched (for the bench's gpu_launches)
        # slot-range passes of the screen: None = planned from the last
        # iteration's postings (screen_passes), an int forces a count (1 = off)
        self.passes = None
        self.last_postings = None
        self._doc_freq = None
        # postings counted from the rows' document frequencies (one pass over
        # the terms per assign); False: in the screen, per object entry — for
        # callers whose rows change every step (the streamed end-to-end paths)
        self.df_counter = True
        self._pass_df = None
        # IVFD (rule 1) in its own loop order: the object-inverted kernel
        # (ivfkm_assign_ivfd); False serves IVFD through the IVF kernels with
        # the IVFD label rule (identical results)
        self.ivfd_native = True
        # slot-range passes stage presorted rows (ivfkm_assign_screen_ex)
        self.presort = True
        self._presort = None
        # sparse spans read through their slot bytes (ivfkm_bivf_slots): None =
        # at large k (>= 16 spans), where they are a sixth of the screen's pairs
        self.sparse_slots = None
        self._slotbuf = [None, None]
        self._xinv = None
        self._ivfd_ws = None

    def _row_order(self, dd):
        """Longest rows first (computed once per dataset, on the device)."""
        order = torch.empty(max(dd.n, 1), dtype=torch.int32, device=self.device)
        ws = torch.empty(int(self.lib.ivfkm_row_order_workspace_size(dd.n)), dtype=torch.uint8,
                         device=self.device)
        _lib.check(self.lib.ivfkm_row_order(dd.n, _p(dd.row_ptr), _p(order), _p(ws), ws.numel(),
                                            _stream()), "ivfkm_row_order")
        return order

    # -- means ---------------------------------------------------------------
    def _rankdir_async(self, dm: DeviceMeans) -> None:
        """Build the rank directory of dm's CSR (ivfkm_rankdir_build) on the
        side stream; assign waits for dm.dir_ready before the rescoring.  The
        one directory buffer is free by then: this runs after the previous
        means' finalize in the current stream's order."""
        dm.dir_ready = None
        if self.side is None or self.rankdir is None:
            return
        cur = torch.cuda.current_stream()
        self.side.wait_stream(cur)
        with torch.cuda.stream(self.side):
            _lib.check(self.lib.ivfkm_rankdir_build(self.k, dm.dim, _p(dm.ptr), _p(dm.terms),
                                                    _p(self.rankdir), _stream()),
                       "ivfkm_rankdir_build")
            dm.dir_ready = torch.cuda.Event()
            dm.dir_ready.record(self.side)
        dm.ptr.record_stream(self.side)
        dm.terms.record_stream(self.side)
        self._dir_of = dm

    def build_bivf(self, dm: DeviceMeans) -> DeviceMeans:
        dev = self.device
        self._rankdir_async(dm)
        dm.headers = torch.empty(int(self.lib.ivfkm_bivf_headers_size(self.k, dm.dim)),
                                 dtype=torch.int32, device=dev)
        # plan (headers; the host learns the exact value counts), then fill —
        # in the same call when this parity's value buffers are big enough
        # (no host round trip between the two), else once more after growing
        totals = self._totals  # (screen values, exact values)
        bits = self.screen_bits
        vdt = torch.float16 if bits == 16 else torch.float32
        buf = self._bvbuf[self._bvpar]
        self._bvpar ^= 1  # the previous means keep their arrays
        rc = self.lib.ivfkm_bivf_plan_fill(
            self.k, dm.dim, 0, self.k, _p(dm.ptr), _p(dm.terms), _p(dm.vals), _p(dm.headers),
            C.c_void_p(totals.ctypes.data), _p(buf["pvs"]) if buf else None,
            buf["pvs"].numel() if buf else 0, bits, _p(buf["pv64"]) if buf else None,
            buf["pv64"].numel() if buf else 0, _p(self.ws_bivf), self.ws_bivf.numel(),
            _p(self.ws_fill), self.ws_fill.numel() if self.ws_fill is not None else 0, _stream())
        filled = rc == 0
        if rc != _lib.IVFKM_E_WORKSPACE:
            _lib.check(rc, "ivfkm_bivf_plan_fill")
        n_s, n_64 = int(totals[0]), int(totals[1])
        if dm.nnz < 0:  # deferred update: the plan counted the postings
            dm.nnz = n_64
            dm.terms, dm.vals = dm.terms[:dm.nnz], dm.vals[:dm.nnz]
        if not filled:
            if buf is None or buf["pvs"].numel() < n_s or buf["pv64"].numel() < n_64:
                buf = {"pvs": torch.empty(int(n_s * 1.25) + 1024, dtype=vdt, device=dev),
                       "pv64": torch.empty(int(n_64 * 1.25) + 1024, dtype=torch.float64,
                                           device=dev)}
                self._bvbuf[self._bvpar ^ 1] = buf
            need = int(self.lib.ivfkm_bivf_fill_workspace_size(self.k, dm.dim, dm.nnz))
            if self.ws_fill is None or self.ws_fill.numel() < need:
                self.ws_fill = torch.empty(int(need * 1.25) + 4096, dtype=torch.uint8, device=dev)
            rc = self.lib.ivfkm_bivf_fill(self.k, dm.dim, 0, self.k, _p(dm.ptr), _p(dm.terms),
                                          _p(dm.vals), _p(dm.headers), _p(buf["pvs"]), bits,
                                          _p(buf["pv64"]), dm.nnz, _p(self.ws_fill),
                                          self.ws_fill.numel(), _stream())
            _lib.check(rc, "ivfkm_bivf_fill")
        dm.pvs = buf["pvs"][:max(n_s, 1)]
        dm.pv64 = buf["pv64"][:max(n_64, 1)]
        dm.screen_bits = bits
        dm.slot8 = None
        use_slots = self.sparse_slots if self.sparse_slots is not None else self.nblk // 8 >= 16
        if use_slots and bits == 16:
            par = self._bvpar ^ 1  # the value buffers' parity of this build
            sb = self._slotbuf[par]
            need = int(self.lib.ivfkm_bivf_slots_size(self.k, dm.dim, n_s))
            if sb is None or sb.numel() < need:
                sb = torch.empty(need + n_s // 4 + 1024, dtype=torch.uint8, device=dev)
                self._slotbuf[par] = sb
            _lib.check(self.lib.ivfkm_bivf_slots(self.k, dm.dim, 0, self.k, _p(dm.ptr),
                                                 _p(dm.terms), _p(dm.headers), _p(sb), _stream()),
                       "ivfkm_bivf_slots")
            dm.slot8 = sb
            self.launches += 2  # span offsets, slot bytes
        # plan: sizes, CUB sort of the k slot keys (single tile / onesweep), perm,
        # mask, count, 2 scans (init + sweep each), offset, nc, {mask, offset}
        # pairs; fill: zero, position keys, CUB onesweep sort of the keys' top
        # 16 bits (histogram, exclusive sum, a pass per 8 bits), write
        nslot = self.nblk * 32
        kbits = max(1, int(np.ceil(np.log2(float(dm.dim) * nslot + 1))))
        self.launches += 11 + (1 if self.k <= 4096 else 6) + 5 + (min(kbits, 16) + 7) // 8
        return dm

    def upload_means(self, ms) -> DeviceMeans:
        return self.build_bivf(DeviceMeans.from_meanset(ms, self.device))

    # -- assign --------------------------------------------------------------
    # postings per object and pass that amortise a pass's per-object cost
    # (row staging, epilogue, state merge); measured on configs 2-4
    PASS_WORK = 95_000

    def screen_passes(self, dm: DeviceMeans) -> int:
        """Slot-range passes for the fp16 screen at large k:
        enough 256-slot spans per pass that an object's pass does about
        PASS_WORK postings, from this assign's V = sum_t no_t * nc_t (object
        document frequencies against the BIVF's per-term posting counts; one
        small reduction and read-back, only at k >= 4,096 where a screen
        takes 100 ms and more)."""
        if self.passes is not None:
            return int(self.passes)
        spans = self.nblk // 8
        if self.screen_bits != 16 or spans < 16 or self.dd.n == 0:
            return 1
        nh = self.dd.dim * self.nblk
        nc = dm.headers[2 * nh + 1:2 * nh + 1 + self.dd.dim].to(torch.float64)
        if self._pass_df is None or self._pass_df[0] is not self.dd.terms:
            self._pass_df = (self.dd.terms, torch.bincount(
                self.dd.terms.long(), minlength=self.dd.dim).to(torch.float64))
        v = float(torch.dot(self._pass_df[1], nc).item())
        w = max(v / (self.dd.n * spans), 1.0)  # postings per (object, span)
        # whole spans per warp: a pass's CTAs run four warps, and 5 or 11 spans
        # leave some of them idle (config 4: 8 spans per pass 5.77 s, 11: 5.94 s,
        # 12: 6.21 s; config 2: 4 spans 115 ms, 5: 168 ms, 3: 139 ms)
        per = max(4, int(self.PASS_WORK / w) // 4 * 4)
        p = int(np.ceil(spans / per))
        return p if p > 1 else 1

    def doc_freq(self) -> torch.Tensor:
        """Objects per term of the current rows (ivfkm_doc_freq; uint32 held as
        int32), computed once per corpus: the screen's posting counter is
        sum_t doc_freq[t] * nc[t] instead of a gather per object entry."""
        dd = self.dd
        if not self.df_counter:
            return None
        if self._doc_freq is None or self._doc_freq[0] is not dd.terms:
            df = torch.empty(dd.dim, dtype=torch.int32, device=self.device)
            _lib.check(self.lib.ivfkm_doc_freq(dd.nnz, _p(dd.terms), dd.dim, _p(df), _stream()),
                       "ivfkm_doc_freq")
            self._doc_freq = (dd.terms, df)
        return self._doc_freq[1]

    def assign(self, dm: DeviceMeans, prev: torch.Tensor | None, events=None,
               rule: int = 0) -> torch.Tensor:
        """Launch the assignment step; returns the (device) 0-based labels.

        ``events``: optional (start, end) torch.cuda.Event pair recorded around
        the screen kernel (the dominant kernel) on the current stream.
        ``rule``: 0 = IVF argmax, 1 = IVFD (argmax only above 0.0, else mean 0;
        see include/ivfkm.h).
        """
        dd = self.dd
        out = self.labels[self.cur]
        if prev is not None and prev.data_ptr() == out.data_ptr():
            self.cur ^= 1
            out = self.labels[self.cur]
        if rule == 1 and self.ivfd_native:
            return self._assign_ivfd(dm, prev, out, events)
        self.lib.ivfkm_set_tuning(self.rowcap, 0, -1)
        npass = self.screen_passes(dm)
        _lib.check(self.lib.ivfkm_set_screen_option(1, npass), "ivfkm_set_screen_option")
        order = self.order if self.order is not None and dd.n == self.order.numel() else None
        st = _stream()
        if events is not None:
            events[0].record()
        ps = self._presort_buffers() if npass > 1 and self.presort else (None, None)
        rc = self.lib.ivfkm_assign_screen_ex(dd.n, _p(dd.row_ptr), _p(dd.terms), _p(dd.val32),
                                             _p(dd.xnorm), self.k, dd.dim, _p(dm.headers),
                                             _p(dm.pvs), dm.screen_bits, _MU_MAX, _p(self.stats),
                                             _p(order), _p(ps[0]), _p(ps[1]),
                                             _p(dm.slot8 if dm.screen_bits == 16 else None),
                                             _p(self.doc_freq()), _p(self.ws_assign),
                                             self.ws_assign.numel(), st)
        _lib.check(rc, "ivfkm_assign_screen_ex")
        if ps[0] is not None:
            self.launches += 1
        self.launches += 1  # the postings counter from the document frequencies
        self.launches += npass - 1
        if events is not None:
            events[1].record()
        if self.rankdir is not None:
            # the directory built on the side stream for these very means, or
            # (another engine's means, a rebuilt buffer) built here
            pre = dm.dir_ready is not None and self._dir_of is dm
            if pre:
                torch.cuda.current_stream().wait_event(dm.dir_ready)
            elif self.side is not None:  # the buffer may still be written for other means
                torch.cuda.current_stream().wait_stream(self.side)
            rc = self.lib.ivfkm_assign_finish_dir(
                dd.n, _p(dd.row_ptr), _p(dd.terms), _p(dd.val64), self.k, dd.dim,
                _p(dm.headers), _p(dm.pv64), _p(dm.ptr), None if pre else _p(dm.terms),
                _p(dm.vals), _p(self.rankdir), _p(prev), _p(out), _p(self.sims), _p(self.sizes),
                _p(self.stats), rule, _p(self.ws_assign), self.ws_assign.numel(), st)
            if not pre:
                self._dir_of = None  # the buffer now holds dm's directory, unmarked
            _lib.check(rc, "ivfkm_assign_finish_dir")
            self.launches += 6  # directory bits + ranks, winner histogram, scan (2), grouping
        else:
            rc = self.lib.ivfkm_assign_finish(dd.n, _p(dd.row_ptr), _p(dd.terms), _p(dd.val64),
                                              self.k, dd.dim, _p(dm.headers), _p(dm.pv64),
                                              _p(prev), _p(out), _p(self.sims), _p(self.sizes),
                                              _p(self.stats), rule, _p(self.ws_assign),
                                              self.ws_assign.numel(), st)
            _lib.check(rc, "ivfkm_assign_finish")
        self.launches += 4
        return out

    def _presort_buffers(self):
        dd = self.dd
        if self._presort is None or self._presort[0] is not dd.terms:
            # per entry {term, dense prefix} and {dense-run start, value}
            self._presort = (dd.terms, torch.empty(2 * max(dd.nnz, 1), dtype=torch.int32,
                                                   device=self.device),
                             torch.empty(2 * max(dd.nnz, 1), dtype=torch.float32,
                                         device=self.device))
        return self._presort[1], self._presort[2]

    IVFD_SLOT_BYTES = 4 << 30  # the wave's per-mean similarity slots (N float64 each)

    def objects_inverted(self):
        """The objects' inverted file (term-major object postings, objects
        ascending within a term) of the current dataset, built once."""
        dd = self.dd
        if self._xinv is not None and self._xinv[0] is dd.terms:
            return self._xinv[1]
        dev = self.device
        x_ptr = torch.empty(dd.dim + 1, dtype=torch.int64, device=dev)
        x_obj = torch.empty(max(dd.nnz, 1), dtype=torch.int32, device=dev)
        x_val = torch.empty(max(dd.nnz, 1), dtype=torch.float64, device=dev)
        ws = torch.empty(int(self.lib.ivfkm_objects_inverted_workspace_size(dd.nnz, dd.dim)),
                         dtype=torch.uint8, device=dev)
        _lib.check(self.lib.ivfkm_objects_inverted(
            dd.n, dd.nnz, dd.dim, _p(dd.row_ptr), _p(dd.terms), _p(dd.val64), _p(x_ptr),
            _p(x_obj), _p(x_val), _p(ws), ws.numel(), _stream()), "ivfkm_objects_inverted")
        self.launches += 5
        self._xinv = (dd.terms, (x_ptr, x_obj, x_val))
        return self._xinv[1]

    def _assign_ivfd(self, dm: DeviceMeans, prev, out, events):
        dd = self.dd
        x_ptr, x_obj, x_val = self.objects_inverted()
        wave = int(max(1, min(self.k, self.IVFD_SLOT_BYTES // max(8 * dd.n, 1))))
        need = int(self.lib.ivfkm_ivfd_workspace_size(dd.n, wave))
        if self._ivfd_ws is None or self._ivfd_ws.numel() < need:
            self._ivfd_ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        if events is not None:
            events[0].record()
        rc = self.lib.ivfkm_assign_ivfd(dd.n, dd.dim, _p(x_ptr), _p(x_obj), _p(x_val), self.k,
                                        _p(dm.ptr), _p(dm.terms), _p(dm.vals), _p(prev), _p(out),
                                        _p(self.sims), _p(self.sizes), _p(self.stats), wave,
                                        _p(self._ivfd_ws), self._ivfd_ws.numel(), _stream())
        _lib.check(rc, "ivfkm_assign_ivfd")
        if events is not None:
            events[1].record()
        self.launches += 2 * ((self.k + wave - 1) // wave) + 2
        return out

    def score_labels(self, dm: DeviceMeans, labels0: torch.Tensor) -> None:
        dd = self.dd
        rc = self.lib.ivfkm_score_labels(dd.n, _p(dd.row_ptr), _p(dd.terms), _p(dd.val64),
                                         self.k, dd.dim, _p(dm.headers), _p(dm.pv64),
                                         _p(labels0), _p(self.sims), _p(self.stats), _stream())
        _lib.check(rc, "ivfkm_score_labels")
        self.launches += 2

    def read_stats(self) -> IterStats:
        self.stats_async()
        torch.cuda.current_stream().synchronize()
        return self.stats_ready()

    def stats_async(self) -> None:
        """Queue the statistics' device->host copy (read with stats_ready after
        any later synchronisation, e.g. the one inside update)."""
        self.stats_host.copy_(self.stats, non_blocking=True)

    def stats_ready(self) -> IterStats:
        raw = _lib.Stats.from_buffer_copy(self.stats_host.numpy().tobytes())
        st = IterStats.from_raw(raw)
        self.last_postings = st.postings
        return st

    # -- update --------------------------------------------------------------
    def update(self, labels0: torch.Tensor, dm: DeviceMeans) -> DeviceMeans:
        """New means from the assignment (sizes must be the ones ivfkm_assign wrote)."""
        dd = self.dd
        out = update_rows(self.lib, dd.n, dd.nnz, dd.row_ptr, dd.terms, dd.val64, labels0,
                          self.sizes, dm, self.k, dd.dim, self.ws_update, self.total_host,
                          self.upd_state, deferred=self._defer_ok(dm))
        self.launches += (delta_update_launches(self.k, dd.dim) if self.upd_state is not None
                          else update_launches(self.k, dd.dim))
        return self.build_bivf(out)

    def _defer_ok(self, dm: DeviceMeans) -> bool:
        """The size read is skipped only while the capacity bound stays small
        (<= 2 GB of mean arrays); at the largest configs the exact size is
        worth its synchronisation."""
        return (self.dd.nnz + dm.nnz) * 12 <= (2 << 30)

    def set_sizes_from_labels(self, labels0: torch.Tensor) -> None:
        """sizes = bincount(labels) for an externally supplied assignment."""
        self.sizes.copy_(torch.bincount(labels0.long(), minlength=self.k))


class HostIteration:
    """One Lloyd iteration through host buffers — the end-to-end path.

    Every call copies the corpus (pinned HostDataset) and the current means
    host -> device, runs assign + update on the GPU, and reads labels, the
    statistics and the new means back into pinned buffers; the returned
    MeanSet wraps those host buffers (double-buffered, so the next call can
    upload them while they stay valid).  Equivalent to the reference's
    assign_ivf + objective_cosine + update_ivf on host arrays.
    """

    def __init__(self, hd: HostDataset, k: int, device="cuda", prefetch: bool = True):
        self.hd, self.k = hd, int(k)
        self.device = torch.device(device)
        self.eng = None
        self.buf = [None, None]
        self.cur = 0
        self.labels_host = torch.empty(hd.n, dtype=torch.int32).pin_memory()
        self.last_h2d = self.last_d2h = 0
        # the next step's corpus upload overlaps this step's kernels on a copy stream
        self.prefetch = prefetch
        self.copy_stream = torch.cuda.Stream(device=self.device) if prefetch else None
        self.next_dd = None
        self.next_ready = None

    def _upload(self):
        with torch.cuda.stream(self.copy_stream):
            dd = DeviceDataset(self.hd, self.device, copies_only=True)
            ev = torch.cuda.Event()
            ev.record(self.copy_stream)
        return dd, ev

    def _host_buffers(self, nnz: int):
        b = self.buf[self.cur]
        if b is None or b["cap"] < nnz:
            # (re)allocate both halves of the double buffer together, with headroom,
            # so steady-state steps never pin memory
            cap = int(nnz * 1.5) + 1024
            for i in (0, 1):
                if self.buf[i] is None or self.buf[i]["cap"] < nnz:
                    if i != self.cur and self.buf[i] is not None:
                        continue  # still referenced by the MeanSet returned last step
                    self.buf[i] = {
                        "cap": cap,
                        "ptr": torch.empty(self.k + 1, dtype=torch.int64).pin_memory(),
                        "terms": torch.empty(cap, dtype=torch.int32).pin_memory(),
                        "vals": torch.empty(cap, dtype=torch.float64).pin_memory(),
                        "ret": torch.empty(self.k, dtype=torch.uint8).pin_memory()}
            b = self.buf[self.cur]
        return b

    def step(self, ms: MeanSet):
        dev = self.device
        if self.prefetch:
            if self.next_dd is None:
                self.next_dd, self.next_ready = self._upload()
            dd, ready = self.next_dd, self.next_ready
        else:
            dd = DeviceDataset(self.hd, dev)  # H2D of the corpus (pinned, async)
        with warnings.catch_warnings():  # read-only views of pinned buffers: only read here
            warnings.simplefilter("ignore", UserWarning)
            t = lambda a: torch.from_numpy(np.asarray(a))  # noqa: E731
            ptr = t(ms.indptr).to(dev, non_blocking=True)
            terms = t(ms.term_ids).to(dev, non_blocking=True) - 1
            vals = t(ms.values).to(dev, non_blocking=True)
            ret = t(np.asarray(ms.retained).view(np.uint8)).to(dev, non_blocking=True)
        if self.prefetch:
            # the means go first on the H2D engine; then the next step's corpus
            # streams in on the copy stream while this step computes
            torch.cuda.current_stream().wait_event(ready)
            dd.finish()
            for t_ in (dd.row_ptr, dd.terms, dd.val64, dd.xnorm, dd.val32):
                t_.record_stream(torch.cuda.current_stream())
            go = torch.cuda.Event()
            go.record()
            self.copy_stream.wait_event(go)
            self.next_dd, self.next_ready = self._upload()
        if self.eng is None:  # after the wait: the engine reads the rows on this stream
            self.eng = LloydEngine(dd, self.k)
            self.eng.df_counter = False  # new rows every step
        self.eng.dd = dd
        dm = self.eng.build_bivf(DeviceMeans(self.k, ms.dim, ptr, terms, vals, ret))
        lab = self.eng.assign(dm, None)
        st = self.eng.read_stats()
        self.labels_host.copy_(lab, non_blocking=True)
        new = self.eng.update(lab, dm)
        self.cur ^= 1
        b = self._host_buffers(new.nnz)
        b["ptr"].copy_(new.ptr, non_blocking=True)
        b["terms"][: new.nnz].copy_(new.terms + 1, non_blocking=True)
        b["vals"][: new.nnz].copy_(new.vals, non_blocking=True)
        b["ret"].copy_(new.retained, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        out = MeanSet.trusted(self.k, ms.dim, "sparse_inverted", b["ptr"].numpy(),
                              b["terms"][: new.nnz].numpy(), b["vals"][: new.nnz].numpy(),
                              b["ret"].numpy().view(np.bool_))
        labels = self.labels_host.numpy() + 1
        self.last_h2d = self.hd.nbytes + ms.indptr.nbytes + ms.term_ids.nbytes + \
            ms.values.nbytes + np.asarray(ms.retained).nbytes
        self.last_d2h = self.labels_host.numel() * 4 + C.sizeof(_lib.Stats) + \
            (self.k + 1) * 8 + new.nnz * 12 + self.k
        return labels, out, st


class StreamIteration:
    """Lloyd iterations with the corpus streamed from pinned host memory every
    step and the step's result read back — labels, objective and counters
    (the per-iteration record of clustering.py:154-176); the means are the
    model state and stay on the device between steps, as inside ``run``.

    The next step's corpus upload overlaps the current step's kernels on a
    copy stream (the H2D engine), the labels come back on the D2H engine.
    """

    def __init__(self, hd: HostDataset, k: int, means: MeanSet, device="cuda"):
        self.hd, self.k = hd, int(k)
        self.device = torch.device(device)
        self.means0 = means
        self.eng = None
        self.dm = None
        self.prev = None
        self.labels_host = torch.empty(hd.n, dtype=torch.int32).pin_memory()
        self.copy_stream = torch.cuda.Stream(device=self.device)
        self.next_dd = None
        self.next_ready = None
        self.last_h2d = self.last_d2h = 0

    def _upload(self):
        with torch.cuda.stream(self.copy_stream):
            dd = DeviceDataset(self.hd, self.device, copies_only=True)
            ev = torch.cuda.Event()
            ev.record(self.copy_stream)
        return dd, ev

    def step(self):
        if self.next_dd is None:
            self.next_dd, self.next_ready = self._upload()
        dd, ready = self.next_dd, self.next_ready
        torch.cuda.current_stream().wait_event(ready)
        dd.finish()  # decode + fp32 cast here, not on the copy stream
        for t_ in (dd.row_ptr, dd.terms, dd.val64, dd.xnorm, dd.val32):
            t_.record_stream(torch.cuda.current_stream())
        go = torch.cuda.Event()
        go.record()
        self.copy_stream.wait_event(go)
        self.next_dd, self.next_ready = self._upload()  # the next step's corpus, in flight
        if self.eng is None:
            self.eng = LloydEngine(dd, self.k)
            self.eng.df_counter = False  # new rows every step
            self.dm = self.eng.upload_means(self.means0)
        self.eng.dd = dd
        lab = self.eng.assign(self.dm, self.prev)
        self.eng.stats_async()  # objective, changed, counters: the step's result
        self.labels_host.copy_(lab, non_blocking=True)
        self.dm = self.eng.update(lab, self.dm)
        self.prev = lab
        torch.cuda.current_stream().synchronize()
        st = self.eng.stats_ready()
        self.last_h2d = self.hd.nbytes
        self.last_d2h = self.labels_host.numel() * 4 + C.sizeof(_lib.Stats)
        return self.labels_host.numpy() + 1, st

