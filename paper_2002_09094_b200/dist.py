"""Multi-GPU IVF Lloyd iteration: objects sharded, means replicated, exact
cluster-range merge (BASELINE.json:north_star).

One process per GPU (torch.distributed, NCCL over NVLink; gloo for the CPU
tests).  Per iteration:

* assign — purely local: every rank screens and rescores its contiguous row
  shard against the replicated means (no communication; the reference's
  per-object independence, _kernels.pyx:116-125).
* statistics — one int64 all-reduce (pack_stats): postings V, changed
  labels, near-ties, overflows, the objective's range flags, the 34 limbs of
  the exact objective accumulator and the k cluster sizes.  Integer sums are
  order-free, so the objective stays the exactly rounded sum (math.fsum
  semantics) for any rank count.
* update — cluster range r = [r*k/P, (r+1)*k/P) is owned by rank r, which
  keeps the rows of every object labelled in its range (``Members``, in
  ascending global object id).  Each iteration only what changed moves
  (ShardComm.exchange_members): a 16-byte notice (gid, new label) to the old
  owner of every object whose label changed, and the row itself to the new
  owner when the owner changed — one count all-to-all, one packed byte
  all-to-all.  The owner drops leavers, relabels stayers and merges arrivals
  by gid, so it sums its clusters' members in ascending global object order:
  its float64 sums, divisions and pairwise norms are bit-identical to the
  single-GPU update (variants.py:254-307) — the means do not depend on P.
  Owners then all-gather their mean slices (one size all-gather, one packed
  byte all-gather) and every rank rebuilds the bitmap-block inverted file.

Raw member rows, not pre-reduced partial sums, are what keeps the float64
summation order — and so the means — independent of the rank count; after
the first iteration the exchange carries only the movers (a few percent of
the rows at steady state) instead of the whole corpus.

The exchange code is device-agnostic (torch tensors + torch.distributed);
the local compute is injected, so tests/test_dist.py runs the same exchange
and statistics packing over gloo on CPU with the oracle as the local compute.
"""

from __future__ import annotations

import json
import os
import sys
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

__all__ = ["shard_rows", "cluster_range", "Rows", "Members", "ShardComm", "DistLloyd",
           "pack_stats", "unpack_stats", "STAT_WORDS", "bench_multi"]


def shard_rows(indptr: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Contiguous row ranges balanced by stored entries (a first-cut estimate
    of assign work; SURVEY.md §8(e) Partitioning)."""
    n = len(indptr) - 1
    w = np.asarray(indptr, dtype=np.int64) + np.arange(n + 1, dtype=np.int64)  # nnz + 1 per row
    total = int(w[-1])
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(w, total * r // world, side="left")))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def cluster_range(k: int, world: int, rank: int) -> tuple[int, int]:
    return rank * k // world, (rank + 1) * k // world


def cluster_owner_bounds(k: int, world: int) -> torch.Tensor:
    return torch.tensor([cluster_range(k, world, r)[1] for r in range(world)], dtype=torch.int64)


@dataclass
class Rows:
    """A CSR block of object rows (0-based terms) with one label per row."""

    row_ptr: torch.Tensor  # int64 [n+1], starting at 0
    terms: torch.Tensor    # int32 [nnz]
    vals: torch.Tensor     # float64 [nnz]
    labels: torch.Tensor   # int32 [n], global 0-based cluster ids

    @property
    def n(self) -> int:
        return int(self.row_ptr.numel() - 1)

    @property
    def nnz(self) -> int:
        return int(self.terms.numel())


@dataclass
class Members(Rows):
    """An owner's member rows: every object labelled in its cluster range, in
    ascending global object id (``gid``) — the order the single-GPU update
    sums them in, so the owner's means do not depend on the rank count."""

    gid: torch.Tensor = None  # int64 [n], ascending


# -- statistics vector (one int64 all-reduce per iteration) -------------------
STAT_WORDS = 5 + 34  # V, changed, near-ties, overflow, objective flags, 34 limbs


def pack_stats(vec: torch.Tensor, raw: torch.Tensor, sizes: torch.Tensor) -> torch.Tensor:
    """Fill ``vec`` (int64 [STAT_WORDS + k]) from an ivfkm_stats block viewed as
    int64 (``raw``: postings, changed, near_ties, overflow, queue_len,
    obj_flags, 34 limbs) and the k cluster sizes.  Integer sums are
    order-free, so the all-reduced objective is still exactly rounded."""
    vec[:4] = raw[:4]
    vec[4] = raw[5]  # obj_flags: a summand outside the accumulator on any rank
    vec[5:STAT_WORDS] = raw[6:40]
    vec[STAT_WORDS:] = sizes
    return vec


def unpack_stats(h) -> dict:
    """The all-reduced vector (host) -> global statistics (raises like
    IterStats.from_raw when any rank saw an objective summand out of range)."""
    from .engine import objective_from_limbs

    h = [int(x) for x in h[:STAT_WORDS]]
    if h[4]:
        raise FloatingPointError("objective summand outside the exact accumulator range")
    return dict(postings=h[0], changed=h[1], near_ties=h[2], overflow=h[3],
                objective=objective_from_limbs(h[5:STAT_WORDS]))


def _bytes(t: torch.Tensor) -> torch.Tensor:
    """A flat byte view (empty tensors may carry a zero stride)."""
    t = t.reshape(-1)
    if t.numel() == 0:
        return torch.empty(0, dtype=torch.uint8, device=t.device)
    return t.contiguous().view(torch.uint8)


def _gather_entries(row_ptr, terms, vals, sel, total: int):
    """The entries of rows ``sel`` (int64 index) of a CSR block, concatenated;
    ``total`` = their count (known on the host: no device read)."""
    dev = row_ptr.device
    lens = row_ptr[sel + 1] - row_ptr[sel]
    ptr = torch.zeros(sel.numel() + 1, dtype=torch.int64, device=dev)
    torch.cumsum(lens, 0, out=ptr[1:])
    seg = torch.repeat_interleave(torch.arange(sel.numel(), device=dev), lens,
                                  output_size=total)
    idx = row_ptr[sel][seg] + (torch.arange(total, device=dev) - ptr[:-1][seg])
    return terms[idx], vals[idx]


class ShardComm:
    """The collectives of one Lloyd iteration over a process group."""

    def __init__(self, rank: int, world: int, group=None):
        self.rank, self.world, self.group = rank, world, group
        self.last_exchange_bytes = 0

    def allreduce_sum_(self, t: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def _a2a_bytes(self, send: torch.Tensor, send_counts: list[int], recv_counts: list[int]):
        out = torch.empty(sum(recv_counts), dtype=torch.uint8, device=send.device)
        if self.world == 1:
            out.copy_(send)
            return out
        dist.all_to_all_single(out, send, recv_counts, send_counts, group=self.group)
        return out

    def plan_exchange(self, local: Rows, prev: torch.Tensor | None, k: int,
                      first: bool) -> dict:
        """The device side of exchange_members, with no host read: which
        local objects send a notice (label changed) or their row (owner
        changed), grouped by destination, and per destination the counts
        [notices, rows, row entries, leavers, leaver entries] — all-to-all'ed
        so every rank also holds what it will receive.  The caller reads
        ``counts``/``rcounts`` together with the iteration's statistics (one
        host read per iteration) and passes them to exchange_members."""
        dev = local.row_ptr.device
        P = self.world
        bounds = cluster_owner_bounds(k, P).to(dev)
        new = local.labels.to(torch.int64)
        new_own = torch.bucketize(new, bounds, right=True)
        n = new.numel()
        if first or prev is None:
            old_own = torch.full_like(new_own, P)  # nobody owns anything yet
            notice = torch.zeros(n, dtype=torch.bool, device=dev)
            mover = torch.ones(n, dtype=torch.bool, device=dev)
        else:
            old_own = torch.bucketize(prev.to(torch.int64), bounds, right=True)
            notice = new != prev.to(torch.int64)
            mover = notice & (new_own != old_own)
        lens = local.row_ptr[1:] - local.row_ptr[:-1]
        key_n = torch.where(notice, old_own, P)
        key_m = torch.where(mover, new_own, P)
        key_l = torch.where(mover & (old_own < P), old_own, P)  # leavers, by old owner
        cnt = torch.zeros(P + 1, 5, dtype=torch.int64, device=dev)
        one = torch.ones(n, dtype=torch.int64, device=dev)
        cnt[:, 0].index_add_(0, key_n, one)
        cnt[:, 1].index_add_(0, key_m, one)
        cnt[:, 2].index_add_(0, key_m, lens)
        cnt[:, 3].index_add_(0, key_l, one)
        cnt[:, 4].index_add_(0, key_l, lens)
        cnt = cnt[:P].contiguous()
        rcnt = torch.empty_like(cnt)
        if P > 1:
            dist.all_to_all_single(rcnt, cnt, group=self.group)
        else:
            rcnt.copy_(cnt)
        return dict(order_n=torch.argsort(key_n, stable=True),
                    order_m=torch.argsort(key_m, stable=True), new=new, lens=lens,
                    counts=cnt, rcounts=rcnt, k=k, first=first or prev is None)

    def exchange_members(self, owned: "Members | None", gid0: int, local: Rows,
                         prev: torch.Tensor | None, k: int, plan: dict | None = None,
                         host_counts=None) -> Members:
        """Bring the cluster owners' member sets up to the new labels.

        Only what changed crosses the wire: for every object whose label
        changed, a 16-byte notice (gid, new label) to its old owner, and —
        when its owner changed too — the row itself (gid, label, length, then
        int32 terms + float64 values) to the new owner; the first iteration
        (``owned is None``) routes every row.  One packed byte all-to-all.
        The owner drops leavers, relabels stayers and merges arrivals by gid,
        so its members stay in ascending global object order.  With ``plan``
        and its ``host_counts`` (plan_exchange; read by the caller together
        with the iteration's statistics) nothing here reads the device: every
        size comes from those counts."""
        dev = local.row_ptr.device
        P, r = self.world, self.rank
        if plan is None:
            plan = self.plan_exchange(local, prev, k, owned is None)
        if host_counts is None:
            host_counts = torch.stack([plan["counts"], plan["rcounts"]]).cpu().tolist()
        sc, rc = host_counts
        bounds = cluster_owner_bounds(k, P).to(dev)
        n_nt = sum(c[0] for c in sc)
        n_mv = sum(c[1] for c in sc)
        e_mv = sum(c[2] for c in sc)
        nt = plan["order_n"][:n_nt]
        mv = plan["order_m"][:n_mv]
        new, lens = plan["new"], plan["lens"]

        def nbytes(c):
            return 16 * c[0] + 24 * c[1] + 4 * c[2] + (4 if c[2] % 2 else 0) + 8 * c[2]

        gid = torch.arange(new.numel(), device=dev, dtype=torch.int64) + gid0
        notes = torch.stack([gid[nt], new[nt]], 1).reshape(-1)
        meta = torch.stack([gid[mv], new[mv], lens[mv]], 1).reshape(-1)
        m_terms, m_vals = _gather_entries(local.row_ptr, local.terms, local.vals, mv, e_mv)
        parts, o_nt, o_mv, o_e = [], 0, 0, 0
        for d in range(P):
            a, b, e = sc[d][0], sc[d][1], sc[d][2]
            parts.append(_bytes(notes[2 * o_nt:2 * (o_nt + a)]))
            parts.append(_bytes(meta[3 * o_mv:3 * (o_mv + b)]))
            t = m_terms[o_e:o_e + e]
            if e % 2:
                t = torch.cat([t, torch.zeros(1, dtype=torch.int32, device=dev)])
            parts.append(_bytes(t))
            parts.append(_bytes(m_vals[o_e:o_e + e]))
            o_nt, o_mv, o_e = o_nt + a, o_mv + b, o_e + e
        send = torch.cat(parts) if parts else torch.zeros(0, dtype=torch.uint8, device=dev)
        recv = self._a2a_bytes(send, [nbytes(c) for c in sc], [nbytes(c) for c in rc])
        self.last_exchange_bytes = int(send.numel())
        # parse, source by source (sources hold ascending, disjoint gid ranges)
        r_notes, r_meta, r_terms, r_vals, off = [], [], [], [], 0
        for src in range(P):
            a, b, e = rc[src][0], rc[src][1], rc[src][2]
            seg = recv[off:off + nbytes(rc[src])]
            q = 0
            r_notes.append(seg[q:q + 16 * a].view(torch.int64).view(-1, 2))
            q += 16 * a
            r_meta.append(seg[q:q + 24 * b].view(torch.int64).view(-1, 3))
            q += 24 * b
            r_terms.append(seg[q:q + 4 * e].view(torch.int32))
            q += 4 * e + (4 if e % 2 else 0)
            r_vals.append(seg[q:q + 8 * e].view(torch.float64))
            off += nbytes(rc[src])
        notes_in = torch.cat(r_notes)
        meta_in = torch.cat(r_meta)
        a_terms = torch.cat(r_terms)
        a_vals = torch.cat(r_vals)
        n_arr = sum(c[1] for c in rc)
        e_arr = sum(c[2] for c in rc)
        a_ptr = torch.zeros(n_arr + 1, dtype=torch.int64, device=dev)
        torch.cumsum(meta_in[:, 2], 0, out=a_ptr[1:])
        a_gid, a_lab = meta_in[:, 0], meta_in[:, 1].to(torch.int32)
        if owned is None:
            return Members(a_ptr, a_terms, a_vals, a_lab, gid=a_gid)
        # the notices: leavers out, stayers relabelled (no data-dependent shapes)
        labels = owned.labels.clone()
        keep = torch.ones(owned.n, dtype=torch.bool, device=dev)
        if notes_in.shape[0]:
            pos = torch.searchsorted(owned.gid, notes_in[:, 0].contiguous())
            nl = notes_in[:, 1]
            stay = torch.bucketize(nl, bounds, right=True) == r
            labels[pos] = torch.where(stay, nl.to(torch.int32), labels[pos])
            keep[pos] = stay
        n_left = sum(c[3] for c in rc)
        e_left = sum(c[4] for c in rc)
        if n_arr == 0 and n_left == 0:
            return Members(owned.row_ptr, owned.terms, owned.vals, labels, gid=owned.gid)
        kept = torch.argsort((~keep).to(torch.int8), stable=True)[:owned.n - n_left]
        # merge kept members and arrivals by gid (both ascending)
        all_gid = torch.cat([owned.gid[kept], a_gid])
        order = torch.argsort(all_gid, stable=True)
        base = owned.terms.numel()
        starts = torch.cat([owned.row_ptr[kept], a_ptr[:-1] + base])[order]
        lens_all = torch.cat([owned.row_ptr[kept + 1] - owned.row_ptr[kept],
                              a_ptr[1:] - a_ptr[:-1]])[order]
        total = owned.nnz - e_left + e_arr
        new_ptr = torch.zeros(all_gid.numel() + 1, dtype=torch.int64, device=dev)
        torch.cumsum(lens_all, 0, out=new_ptr[1:])
        seg = torch.repeat_interleave(torch.arange(all_gid.numel(), device=dev), lens_all,
                                      output_size=total)
        idx = starts[seg] + (torch.arange(total, device=dev) - new_ptr[:-1][seg])
        terms = torch.cat([owned.terms, a_terms])[idx]
        vals = torch.cat([owned.vals, a_vals])[idx]
        all_lab = torch.cat([labels[kept], a_lab])[order]
        return Members(new_ptr, terms, vals, all_lab, gid=all_gid[order])

    def allgather_means(self, ptr: torch.Tensor, terms: torch.Tensor, vals: torch.Tensor,
                        retained: torch.Tensor):
        """Concatenate every rank's mean slice in rank (= cluster) order: one
        size all-gather, then one packed byte all-gather (NCCL: per-rank
        exact sizes; gloo: padded to the largest slice)."""
        if self.world == 1:
            return ptr, terms, vals, retained
        dev = ptr.device
        kl = int(ptr.numel() - 1)
        nl = int(terms.numel())
        cnt = ptr[1:] - ptr[:-1]

        def nb(kl_, nl_):
            return 8 * kl_ + 4 * nl_ + (4 if nl_ % 2 else 0) + 8 * nl_ + kl_

        t = terms if nl % 2 == 0 else torch.cat([terms, torch.zeros(1, dtype=torch.int32,
                                                                     device=dev)])
        buf = torch.cat([_bytes(cnt), _bytes(t), _bytes(vals), _bytes(retained.to(torch.uint8))])
        sz = torch.tensor([kl, nl], dtype=torch.int64, device=dev)
        sizes = [torch.empty_like(sz) for _ in range(self.world)]
        dist.all_gather(sizes, sz, group=self.group)
        sizes = [tuple(x.cpu().tolist()) for x in sizes]
        lens = [nb(a, b) for a, b in sizes]
        if dist.get_backend(self.group) == "nccl":
            outs = [torch.empty(L, dtype=torch.uint8, device=dev) for L in lens]
            dist.all_gather(outs, buf, group=self.group)  # uneven sizes
        else:
            mx = max(lens)
            pad = torch.zeros(mx, dtype=torch.uint8, device=dev)
            pad[:buf.numel()] = buf
            outs = [torch.empty(mx, dtype=torch.uint8, device=dev) for _ in lens]
            dist.all_gather(outs, pad, group=self.group)
        cnts, tl, vl, rl = [], [], [], []
        for (a, b), o in zip(sizes, outs):
            q = 0
            cnts.append(o[q:q + 8 * a].view(torch.int64))
            q += 8 * a
            tl.append(o[q:q + 4 * b].view(torch.int32))
            q += 4 * b + (4 if b % 2 else 0)
            vl.append(o[q:q + 8 * b].view(torch.float64))
            q += 8 * b
            rl.append(o[q:q + a])
        cnt_all = torch.cat(cnts)
        full_ptr = torch.zeros(cnt_all.numel() + 1, dtype=torch.int64, device=dev)
        torch.cumsum(cnt_all, 0, out=full_ptr[1:])
        return full_ptr, torch.cat(tl), torch.cat(vl), torch.cat(rl)


class DistLloyd:
    """One rank of a sharded Lloyd run on the B200 kernels."""

    def __init__(self, ds, k: int, comm: ShardComm, device):
        from .engine import DeviceDataset, HostDataset, LloydEngine

        self.comm, self.k = comm, int(k)
        self.bounds = shard_rows(ds.indptr, comm.world)
        lo, hi = self.bounds[comm.rank]
        ip = np.asarray(ds.indptr)
        a, b = int(ip[lo]), int(ip[hi])

        class _Shard:
            dim = ds.dim
            indptr = ip[lo:hi + 1] - a
            term_ids = np.asarray(ds.term_ids)[a:b]
            values = np.asarray(ds.values)[a:b]

        self.lo, self.hi = lo, hi
        self.host = HostDataset(_Shard, pin=torch.cuda.is_available())
        self.dd = DeviceDataset(self.host, device)
        self.members = None  # this rank's cluster-range member rows (exchange_members)
        self.prev_labels = None
        self._plan = None    # (labels, exchange plan, host counts) from assign
        # the sharded update routes rows to cluster owners and runs the
        # stateless count (no label-delta state, no whole-shard workspace)
        self.eng = LloydEngine(self.dd, self.k, delta_update=False, update_ws=False)
        self.device = self.dd.device
        self.stats_vec = torch.zeros(STAT_WORDS + self.k, dtype=torch.int64, device=self.device)
        self.ws = None  # update workspace of the routed rows, grown on demand

    def assign(self, dm, prev, events=None):
        """Local assign + the one statistics all-reduce; returns labels and
        global (postings, changed, near_ties, overflow, objective, sizes)."""
        lab = self.eng.assign(dm, prev, events=events)
        raw = self.eng.stats.view(torch.int64)  # 6 + 34 words (ivfkm_stats)
        # the update's exchange plan rides on the statistics' host read: one
        # device->host read per iteration for both
        dd = self.dd
        plan = self.comm.plan_exchange(Rows(dd.row_ptr, dd.terms, dd.val64, lab),
                                       self.prev_labels, self.k, self.members is None)
        v = pack_stats(self.stats_vec, raw, self.eng.sizes)
        self.comm.allreduce_sum_(v)
        h = torch.cat([v, raw[:1], plan["counts"].reshape(-1), plan["rcounts"].reshape(-1)]).cpu()
        nv = v.numel()
        self.local_postings = int(h[nv])  # this rank's share (roofline)
        P = self.comm.world
        c = h[nv + 1:].view(2, P, 5).tolist()
        self._plan = (lab, plan, c)
        self.eng.sizes.copy_(v[STAT_WORDS:])  # global sizes for the update
        return lab, unpack_stats(h[:nv])

    def update(self, lab, dm):
        from .engine import DeviceMeans, update_rows

        dd, k = self.dd, self.k
        rows = Rows(dd.row_ptr, dd.terms, dd.val64, lab)
        plan = host = None
        if self._plan is not None and self._plan[0] is lab:
            _, plan, host = self._plan
        recv = self.members = self.comm.exchange_members(self.members, self.lo, rows,
                                                         self.prev_labels, k, plan, host)
        self._plan = None
        self.prev_labels = lab.clone()
        clo, chi = cluster_range(k, self.comm.world, self.comm.rank)
        kl = chi - clo
        if kl > 0:
            p0 = int(dm.ptr[clo])
            p1 = int(dm.ptr[chi])
            prev = DeviceMeans(kl, dd.dim, dm.ptr[clo:chi + 1] - p0, dm.terms[p0:p1],
                               dm.vals[p0:p1], dm.retained[clo:chi])
            need = int(self.eng.lib.ivfkm_update_workspace_size(recv.n, recv.nnz, kl, dd.dim))
            if self.ws is None or self.ws.numel() < need:
                self.ws = torch.empty(int(need * 1.25) + 4096, dtype=torch.uint8,
                                      device=self.device)
            sl = update_rows(self.eng.lib, recv.n, recv.nnz, recv.row_ptr, recv.terms,
                             recv.vals, recv.labels - clo, self.eng.sizes[clo:chi].contiguous(),
                             prev, kl, dd.dim, self.ws)
            parts = (sl.ptr, sl.terms, sl.vals, sl.retained)
        else:
            dev = self.device
            parts = (torch.zeros(1, dtype=torch.int64, device=dev),
                     torch.zeros(0, dtype=torch.int32, device=dev),
                     torch.zeros(0, dtype=torch.float64, device=dev),
                     torch.zeros(0, dtype=torch.uint8, device=dev))
        ptr, terms, vals, ret = self.comm.allgather_means(*parts)
        return self.eng.build_bivf(DeviceMeans(k, dd.dim, ptr, terms, vals, ret))


def bench_multi(args, rank: int, world: int) -> None:
    """bench.py --gpus N under torchrun: strong scaling of one Lloyd run over N
    ranks (objects sharded, means replicated), plus the same metric end to end
    (every step re-uploads each rank's shard from pinned host memory and reads
    the labels and statistics back; the means stay on the devices)."""
    from . import synth
    from .clustering import init_means
    from .engine import DeviceDataset

    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # NCCL writes its version / debug lines to stdout: keep stdout for the one
    # JSON line (bench.py's contract) and send everything before it to stderr
    sys.stdout.flush()
    stdout_fd = os.dup(1)
    os.dup2(2, 1)
    if os.environ.get("MASTER_ADDR") is None:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29513")
    dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    comm = ShardComm(rank, world)
    c = synth.CONFIGS[args.config]
    spec = c["corpus"]
    ds = synth.make_dataset(spec)
    k = c["k"]
    run = DistLloyd(ds, k, comm, dev)
    dm = run.eng.upload_means(init_means(ds, k, c["seed"], representation="sparse_inverted"))
    prev = None
    for _ in range(args.warmup):
        lab, st = run.assign(dm, prev)
        dm = run.update(lab, dm)
        prev = lab
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    posts, local_posts = [], []
    launches0 = run.eng.launches
    clk = None
    if rank == 0:
        sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
        from bench import Clocks  # the driver's nvidia-smi sampler (bench.py)

        clk = Clocks(local)
    s.record()
    for i in range(args.steps):
        lab, st = run.assign(dm, prev, events=ev[i])
        posts.append(st["postings"])
        local_posts.append(run.local_postings)
        dm = run.update(lab, dm)
        prev = lab
    e.record()
    torch.cuda.synchronize()
    clocks = clk.stop() if clk is not None else None
    launches = run.eng.launches - launches0
    ms = torch.tensor([s.elapsed_time(e)], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    screen_s = sum(a.elapsed_time(b) for a, b in ev) / len(ev) / 1000.0
    # roofline of the screen on the slowest rank: its own shard's bytes / time
    from bench import algorithmic_bytes, roofline

    mine = algorithmic_bytes(sum(local_posts) / len(local_posts), run.dd.nnz, run.dd.n,
                             run.eng.screen_bits // 8)
    rl = torch.tensor([mine / screen_s / 1e9], dtype=torch.float64, device=dev)
    slow = rl.clone()
    dist.all_reduce(slow, op=dist.ReduceOp.MIN)  # lowest achieved GB/s over ranks
    # ---- end to end, as the single-GPU e2e leg (engine.StreamIteration): every
    # step re-uploads this rank's shard from pinned host memory and reads the
    # step's result back — labels and the statistics (already a host read of
    # assign) — while the means and the owners' member rows, the model state,
    # stay on the devices
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else max(1, min(args.steps, 3))
    lab_host = torch.empty(run.dd.n, dtype=torch.int32).pin_memory()
    h2d = d2h = 0
    run.eng.df_counter = False  # new rows every step
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        run.dd = DeviceDataset(run.host, dev)
        run.eng.dd = run.dd
        lab, _ = run.assign(dm, prev)
        lab_host.copy_(lab, non_blocking=True)
        dm = run.update(lab, dm)
        prev = lab
        torch.cuda.current_stream().synchronize()
        h2d = run.host.nbytes
        d2h = lab_host.numel() * 4 + (STAT_WORDS + k) * 8
    torch.cuda.synchronize()
    e2e_t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    dist.barrier()
    t = float(ms.item())
    slow_gbs = float(slow[0].item())
    e2e_s = float(e2e_t.item())
    dist.destroy_process_group()
    sys.stdout.flush()
    os.dup2(stdout_fd, 1)
    os.close(stdout_fd)
    if rank == 0:
        # the slowest rank's screen: its algorithmic bytes over its time
        rf = roofline(slow_gbs * screen_s * 1e9, screen_s, None, run.eng.screen_bits)
        rf["per"] = "slowest rank's screen over its shard"

        print(json.dumps({
            "metric": "Lloyd iterations/sec and assign-step postings/sec (% roofline), 1/2/4/8 B200",
            "value": args.steps / (t / 1000.0), "unit": "iter/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "screen": f"fp{run.eng.screen_bits} values, fp32 FMA, rigorous window -> exact f64 rescoring",
            "config": {"workload": f"config{args.config}", "N": ds.n, "D": ds.dim, "k": k,
                       "sum_nnz": int(ds.sum_nnz),
                       "parallelism": f"objects sharded over {world} GPUs, means replicated",
                       "l2": "inputs larger than L2"},
            "postings_per_sec": sum(posts) / (t / 1000.0),
            "roofline": rf,
            "gpu_launches": launches * world,
            "clocks": clocks,
            "e2e": {"value": e2e_steps / e2e_s, "unit": "iter/s",
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "steps": e2e_steps, "per_rank_bytes": True},
            "time": time.strftime("%Y-%m-%dT%H:%M:%S"),
        }), flush=True)
