"""Multi-GPU IVF Lloyd iteration: objects sharded, means replicated, exact
cluster-range merge (BASELINE.json:north_star).

One process per GPU (torch.distributed, NCCL over NVLink; gloo for the CPU
tests).  Per iteration:

* assign — purely local: every rank screens and rescores its contiguous row
  shard against the replicated means (no communication; the reference's
  per-object independence, _kernels.pyx:116-125).
* statistics — one all-reduce of int64: postings V, changed labels,
  near-ties, the 34 limbs of the exact objective accumulator and the k
  cluster sizes.  Integer sums are order-free, so the objective stays the
  exactly rounded sum (math.fsum semantics) for any rank count.
* update — cluster range r = [r*k/P, (r+1)*k/P) is owned by rank r.  Every
  rank routes each of its object rows to the owner of its label
  (all-to-all-v of labels, row lengths, term ids and float64 values).  The
  owner receives its clusters' members from ranks 0..P-1 in rank order, i.e.
  in ascending global object order, so its per-(cluster, term) float64 sums,
  divisions and pairwise norms are bit-identical to the single-GPU update
  (variants.py:254-307) — means do not depend on P.  Owners then
  all-gather their mean slices (sizes first, then padded payloads) and every
  rank rebuilds the bitmap-block inverted file locally.

Raw rows cross NVLink once per iteration (sum_nnz * 12 B in total; ~5.8 GB at
config 3, milliseconds at ~770 GB/s per GPU) instead of pre-reduced partial
sums: that is what keeps the float64 summation order, and hence the means,
independent of the rank count.

The exchange code is device-agnostic (torch tensors + torch.distributed);
the local compute is injected, so tests/test_dist.py runs the same exchange
over gloo on CPU with the oracle as the local compute.
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

__all__ = ["shard_rows", "cluster_range", "Rows", "ShardComm", "DistLloyd", "bench_multi"]


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


class ShardComm:
    """The collectives of one Lloyd iteration over a process group."""

    def __init__(self, rank: int, world: int, group=None):
        self.rank, self.world, self.group = rank, world, group

    def allreduce_sum_(self, t: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def _a2a(self, send: torch.Tensor, send_counts: list[int], recv_counts: list[int]):
        out = torch.empty(sum(recv_counts), dtype=send.dtype, device=send.device)
        if self.world == 1:
            out.copy_(send)
            return out
        dist.all_to_all_single(out, send.contiguous(), recv_counts, send_counts, group=self.group)
        return out

    def route_rows(self, rows: Rows, k: int) -> Rows:
        """Send each row to the owner of its label's cluster range; the result
        holds the owner's rows in ascending global object order."""
        if self.world == 1:  # the only rank owns every cluster: nothing moves
            return rows
        dev = rows.row_ptr.device
        bounds = cluster_owner_bounds(k, self.world).to(dev)
        lab = rows.labels.to(torch.int64)
        owner = torch.bucketize(lab, bounds, right=True)
        order = torch.argsort(owner, stable=True)
        nnz_row = (rows.row_ptr[1:] - rows.row_ptr[:-1])
        obj_cnt = torch.bincount(owner, minlength=self.world)
        ent_cnt = torch.zeros(self.world, dtype=torch.int64, device=dev)
        ent_cnt.index_add_(0, owner, nnz_row)
        counts = torch.stack([obj_cnt, ent_cnt], 1).reshape(-1)
        rcounts = torch.empty_like(counts)
        if self.world > 1:
            dist.all_to_all_single(rcounts, counts, group=self.group)
        else:
            rcounts.copy_(counts)
        c = counts.view(-1, 2).cpu().tolist()
        rc = rcounts.view(-1, 2).cpu().tolist()
        # entries in the routed order
        sel_len = nnz_row[order]
        starts = rows.row_ptr[:-1][order]
        seg = torch.repeat_interleave(torch.arange(order.numel(), device=dev), sel_len)
        seg_start = torch.cumsum(sel_len, 0) - sel_len
        ent_idx = starts[seg] + (torch.arange(seg.numel(), device=dev) - seg_start[seg])
        meta = torch.stack([lab[order], sel_len], 1).reshape(-1)
        r_meta = self._a2a(meta, [2 * a for a, _ in c], [2 * a for a, _ in rc]).view(-1, 2)
        r_terms = self._a2a(rows.terms[ent_idx], [b for _, b in c], [b for _, b in rc])
        r_vals = self._a2a(rows.vals[ent_idx], [b for _, b in c], [b for _, b in rc])
        ptr = torch.zeros(r_meta.shape[0] + 1, dtype=torch.int64, device=dev)
        torch.cumsum(r_meta[:, 1], 0, out=ptr[1:])
        return Rows(ptr, r_terms.to(torch.int32), r_vals, r_meta[:, 0].to(torch.int32))

    def allgather_means(self, ptr: torch.Tensor, terms: torch.Tensor, vals: torch.Tensor,
                        retained: torch.Tensor):
        """Concatenate every rank's mean slice in rank (= cluster) order."""
        if self.world == 1:
            return ptr, terms, vals, retained
        dev = ptr.device
        kl = int(ptr.numel() - 1)
        nl = int(terms.numel())
        sz = torch.tensor([kl, nl], dtype=torch.int64, device=dev)
        sizes = [torch.empty_like(sz) for _ in range(self.world)]
        dist.all_gather(sizes, sz, group=self.group)
        sizes = [tuple(x.cpu().tolist()) for x in sizes]
        kmax = max(a for a, _ in sizes)
        nmax = max(max(b for _, b in sizes), 1)

        def gather(t, length, fill_dtype):
            buf = torch.zeros(length, dtype=fill_dtype, device=dev)
            buf[: t.numel()] = t
            outs = [torch.empty_like(buf) for _ in range(self.world)]
            dist.all_gather(outs, buf, group=self.group)
            return outs

        g_cnt = gather(ptr[1:] - ptr[:-1], kmax, torch.int64)
        g_terms = gather(terms, nmax, torch.int32)
        g_vals = gather(vals, nmax, torch.float64)
        g_ret = gather(retained.to(torch.int32), kmax, torch.int32)
        cnt = torch.cat([g_cnt[r][: sizes[r][0]] for r in range(self.world)])
        full_ptr = torch.zeros(cnt.numel() + 1, dtype=torch.int64, device=dev)
        torch.cumsum(cnt, 0, out=full_ptr[1:])
        full_terms = torch.cat([g_terms[r][: sizes[r][1]] for r in range(self.world)])
        full_vals = torch.cat([g_vals[r][: sizes[r][1]] for r in range(self.world)])
        full_ret = torch.cat([g_ret[r][: sizes[r][0]] for r in range(self.world)]).to(torch.uint8)
        return full_ptr, full_terms, full_vals, full_ret


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
        # the sharded update routes rows to cluster owners and runs the
        # stateless count (no label-delta state, no whole-shard workspace)
        self.eng = LloydEngine(self.dd, self.k, delta_update=False, update_ws=False)
        self.device = self.dd.device
        self.stats_vec = torch.zeros(5 + 34 + self.k, dtype=torch.int64, device=self.device)
        self.ws = None  # update workspace of the routed rows, grown on demand

    def assign(self, dm, prev, events=None):
        """Local assign + the one statistics all-reduce; returns labels and
        global (postings, changed, near_ties, overflow, objective, sizes)."""
        from .engine import objective_from_limbs

        lab = self.eng.assign(dm, prev, events=events)
        raw = self.eng.stats.view(torch.int64)  # 6 + 34 words (ivfkm_stats)
        v = self.stats_vec
        v[:4] = raw[:4]
        v[4] = raw[5]  # obj_flags: nonzero on any rank poisons the objective
        v[5:39] = raw[6:40]
        v[39:] = self.eng.sizes
        self.comm.allreduce_sum_(v)
        h = v.cpu()
        self.local_postings = int(raw[0].item())  # this rank's share (roofline)
        self.eng.sizes.copy_(v[39:])  # global sizes for the update
        if int(h[4]):
            raise FloatingPointError("objective summand outside the exact accumulator range")
        return lab, dict(postings=int(h[0]), changed=int(h[1]), near_ties=int(h[2]),
                         overflow=int(h[3]), objective=objective_from_limbs(h[5:39].tolist()))

    def update(self, lab, dm):
        from .engine import DeviceMeans, update_rows

        dd, k = self.dd, self.k
        rows = Rows(dd.row_ptr, dd.terms, dd.val64, lab)
        recv = self.comm.route_rows(rows, k)
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
    (every step re-uploads each rank's shard and the means from pinned host
    memory and reads labels + means back)."""
    from . import synth
    from .clustering import init_means
    from .engine import DeviceDataset, DeviceMeans

    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
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
    from bench import algorithmic_bytes, measured_peak_hbm

    mine = algorithmic_bytes(sum(local_posts) / len(local_posts), run.dd.nnz, run.dd.n,
                             run.eng.screen_bits // 8)
    rl = torch.tensor([mine / screen_s / 1e9, screen_s], dtype=torch.float64, device=dev)
    slow = rl.clone()
    dist.all_reduce(slow, op=dist.ReduceOp.MIN)  # lowest achieved GB/s over ranks
    # ---- end to end: host buffers in and out every step
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else max(1, min(args.steps, 3))
    host = {name: getattr(dm, name).cpu().pin_memory() for name in ("ptr", "terms", "vals",
                                                                     "retained")}
    lab_host = torch.empty(run.dd.n, dtype=torch.int32).pin_memory()
    h2d = d2h = 0
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        run.dd = DeviceDataset(run.host, dev)
        run.eng.dd = run.dd
        dmh = DeviceMeans(k, ds.dim, host["ptr"].to(dev, non_blocking=True),
                          host["terms"].to(dev, non_blocking=True),
                          host["vals"].to(dev, non_blocking=True),
                          host["retained"].to(dev, non_blocking=True))
        dmh = run.eng.build_bivf(dmh)
        lab, _ = run.assign(dmh, None)
        lab_host.copy_(lab, non_blocking=True)
        new = run.update(lab, dmh)
        host = {name: getattr(new, name).cpu() for name in ("ptr", "terms", "vals", "retained")}
        h2d = run.host.nbytes + sum(v.numel() * v.element_size() for v in host.values())
        d2h = lab_host.numel() * 4 + sum(v.numel() * v.element_size() for v in host.values())
    torch.cuda.synchronize()
    e2e_t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    dist.barrier()
    if rank == 0:
        t = float(ms.item())
        peak, peak_kind = measured_peak_hbm()
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
            "roofline": {"bound": "hbm", "achieved": float(slow[0].item()), "peak": peak,
                         "unit": "GB/s", "frac": float(slow[0].item()) / peak, "traffic": None,
                         "peak_source": peak_kind, "per": "slowest rank's screen over its shard",
                         "kernel": f"screen_kernel (BIVF register screen, fp{run.eng.screen_bits} values)"},
            "gpu_launches": launches * world,
            "clocks": clocks,
            "e2e": {"value": e2e_steps / float(e2e_t.item()), "unit": "iter/s",
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "steps": e2e_steps, "per_rank_bytes": True},
            "time": time.strftime("%Y-%m-%dT%H:%M:%S"),
        }), flush=True)
    dist.destroy_process_group()
