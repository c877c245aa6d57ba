#!/usr/bin/env python
"""Benchmark of the B200 IVF spherical k-means Lloyd path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A *step* is one Lloyd iteration over the whole (synthetic) corpus: assign
(fp16 register screen + exact fp64 rescoring, changed-label count, sizes,
exact objective), the host-side convergence read, and the update (bit-exact
means + bitmap-block inverted-file rebuild).  Default workload is
BASELINE.json configs[1] (N=300k, D=100k, k=1000: the config its metric is
quoted on for one GPU, and one whose reference arm runs real full-size
iterations within the driver's time); ``--config 0..4`` picks another.
Prints ONE JSON line (rank 0).

``value``     Lloyd iterations/s with the corpus resident in HBM (CUDA events on
              the launching stream, barrier + synchronize on both sides, max
              over ranks);
``e2e``       the same metric through host buffers: every step copies the
              corpus host->device from pinned memory and reads the step's result
              (labels, objective, counters) back; ``e2e.run_api`` times the
              public API itself — ``run("IVF", ds, k, seed, max_iter)`` on a
              host Dataset (upload, seeding, per-iteration labels and records);
``roofline``  the screen kernel (dominant): algorithmic bytes of an assign pass
              in this layout over its average
              launch time, against the measured L2 read bandwidth (the
              algorithmic bytes exceed what HBM could deliver: most postings are
              L2 hits, so L2 is the binding ceiling); ``traffic`` / ``l2`` are the
              DRAM and L2->SM bytes ncu measured for the same kernel in this run
              (a one-launch ncu probe of the same commit and iteration);
``secondary`` config 3 (N=8.2M, k=10,000: the largest single-GPU config, one of
              the metric's 1/2/4/8-GPU configs) measured in the same run;
``cpu_baseline`` the reference's own compiled kernel (oracle/_ref) on this host's
              cores over a bounded row sample at the GPU's iteration state,
              plus the numpy update and objective (test infrastructure, used
              here only as the baseline).

``--impl reference`` times the reference CPU path as the reference arm: real
full-corpus Lloyd iterations (the reference kernel on all host threads + the
update and objective), from the same initial means and warm-up as ours.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import re
import shutil
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Lloyd iterations/sec and assign-step postings/sec (% roofline), 1/2/4/8 B200"
UNIT = "iter/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--secondary-config", type=int, default=3)
    ap.add_argument("--no-traffic", action="store_true",
                    help="skip the one-launch ncu probe of DRAM / L2 bytes")
    ap.add_argument("--probe", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--dist", action="store_true",
                    help="use the sharded multi-GPU driver even at one rank (torchrun)")
    ap.add_argument("--cpu-seconds", type=float, default=8.0,
                    help="target CPU time of the sampled assign in the baseline")
    return ap.parse_args()


# ----------------------------------------------------------------- helpers

def measured_peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def l2_peak():
    """The L2->SM read bandwidth tools/l2_peak.cu measured on this pool's
    B200s (profiles/l2_peak.json; MEASURED_PEAKS.json has no L2 figure)."""
    try:
        pk = json.loads((ROOT / "profiles" / "l2_peak.json").read_text())
        return (max(r["GB_per_s"] for r in pk["results"] if r["buffer_mb"] * 2**20 < pk["l2_bytes"]),
                "measured (tools/l2_peak.cu, profiles/l2_peak.json)")
    except Exception:
        return None, None


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def csrc_digest() -> str:
    """Identity of the kernels (sources + ABI header) for stamping profiles."""
    h = hashlib.sha256()
    csrc = ROOT / "paper_2002_09094_b200" / "csrc"
    for p in sorted(list(csrc.glob("*.cu")) + list(csrc.glob("*.cuh")) + list(csrc.glob("*.cpp"))
                    + [ROOT / "include" / "ivfkm.h"]):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()[:16]


def workload(cfg_index):
    from paper_2002_09094_b200 import synth

    c = synth.CONFIGS[cfg_index]
    return c, c["corpus"]


def config_dict(cfg_index, c, spec, ds, world):
    return {
        "workload": f"config{cfg_index}",
        "N": ds.n, "D": ds.dim, "k": c["k"], "sum_nnz": int(ds.sum_nnz),
        "rows": f"{spec.nnz_kind}(mean {spec.nnz_mean:g}"
                + (f", sigma {spec.nnz_sigma:g}" if spec.nnz_kind == "lognormal" else "")
                + f") clipped [{spec.nnz_lo},{spec.nnz_hi}]",
        "terms": f"Zipf(s={spec.zipf_s:g}) without replacement", "values": "tf-idf, L2-normalised",
        "data_seed": spec.seed, "mean_seed": c["seed"],
        "l2": ("inputs larger than L2 (object CSR {:.2f} GB > 126 MB L2)"
               if ds.sum_nnz * 16 > 126e6 else
               "inputs smaller than L2 (object CSR {:.3f} GB), no flush").format(
                   ds.sum_nnz * 16 / 1e9),
        "parallelism": "objects sharded, means replicated" if world > 1 else "single GPU",
    }


class Clocks:
    """Clock / throttle sampler for the timed region (B200_PROFILING.md clocks
    line): NVML every 5 ms from a thread (so even a 0.2 s region gets dozens
    of samples), nvidia-smi -lms 200 when NVML is unavailable."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index=0):
        self.p = self.thread = None
        self.sm, self.mx, self.reasons = [], 0.0, set()
        try:
            import threading

            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(index)
            bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
            self.mx = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            self.stop_flag = threading.Event()

            def run():
                while not self.stop_flag.is_set():
                    self.sm.append(float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)))
                    r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.reasons.update(nm for nm, b in bits.items() if r & b)
                    self.stop_flag.wait(0.005)

            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.thread = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.thread is not None:
            self.stop_flag.set()
            self.thread.join(timeout=5)
            if not self.sm:
                return None
            return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.mx,
                    "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml"}
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [r.split(",") for r in Path(self.f.name).read_text().strip().splitlines() if r]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for nm, val in zip(self.NAMES, r[5:9]):
                    if val.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi"}


def algorithmic_bytes(postings, sum_nnz, n, value_bytes):
    """SURVEY.md §8(d) for this layout: every posting's screen value once
    (b_p = value_bytes: 2 for fp16, 4 for fp32; the bitmap costs 1 bit per
    slot and is not charged), the object entries (int32 term + fp32 value) and
    their three per-term lookups (nc, dense prefix, run start: 12 B), row
    offsets (int64) and the per-object outputs (label + queue slot)."""
    return value_bytes * postings + 20 * sum_nnz + 8 * (n + 1) + 8 * n


# ----------------------------------------------------------------- traffic (ncu)

TRAFFIC_METRICS = ("dram__bytes_read.sum", "dram__bytes_write.sum",
                   "lts__t_sectors_srcunit_tex_op_read.sum")


def ncu_path():
    for p in (shutil.which("ncu"), "/usr/local/cuda/bin/ncu"):
        if p and Path(p).exists():
            return p
    return None


def traffic_probe(cfg, warmup, timeout=300):
    """DRAM and L2->SM bytes of the screen of the first timed iteration —
    summed over its launches (one, or one per slot-range pass) — measured by
    ncu on a child process that replays this run's state (same corpus, seed
    and warm-up: the iterations are deterministic) and marks that assign with
    an NVTX range."""
    ncu = ncu_path()
    if ncu is None:
        return None, "ncu not found"
    cmd = [ncu, "--metrics", ",".join(TRAFFIC_METRICS), "--nvtx", "--nvtx-include", "probe/",
           "-k", "regex:screen_kernel", "--launch-count", "4096", "--csv", "--print-units", "base",
           sys.executable, str(ROOT / "bench.py"), "--probe", "--config", str(cfg),
           "--warmup", str(warmup)]
    try:
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    except Exception as exc:
        return None, f"ncu probe failed: {exc!r}"
    vals, launches = {}, set()
    for line in res.stdout.splitlines():
        cells = [c.strip().strip('"') for c in line.split('","')]
        if len(cells) < 3:
            continue
        for m in TRAFFIC_METRICS:
            if m in cells:
                i = cells.index(m)
                try:
                    unit, v = cells[i + 1], float(cells[i + 2].replace(",", ""))
                except (IndexError, ValueError):
                    continue
                mult = {"byte": 1, "sector": 32}.get(unit, 1)
                vals[m] = vals.get(m, 0.0) + v * mult
                launches.add(cells[0])
    if len(vals) < 3:
        return None, f"ncu probe: no metrics (rc {res.returncode}): {res.stderr[-300:]}"
    return {"dram_bytes": vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"],
            "l2_read_bytes": vals["lts__t_sectors_srcunit_tex_op_read.sum"],
            "launches": len(launches),
            "source": "ncu " + " ".join(cmd[1:14]) + " (this run)"}, None


def stamped_traffic(cfg):
    """profiles/traffic.json's entry for the config, only when it was captured
    from the kernels of this exact source tree (stamp = csrc_digest())."""
    try:
        tr = json.loads((ROOT / "profiles" / "traffic.json").read_text()).get(f"config{cfg}")
    except Exception:
        return None
    if isinstance(tr, dict) and tr.get("csrc") == csrc_digest():
        return dict(tr, source=tr.get("source", "profiles/traffic.json") + " (stamped, same sources)")
    return None


def roofline(avg_b, screen_s, traffic, screen_bits):
    hbm, hbm_src = measured_peak_hbm()
    l2pk, l2_src = l2_peak()
    ach = avg_b / screen_s / 1e9
    r = {"kernel": f"screen_kernel (BIVF register screen, fp{screen_bits} values)",
         "bytes_per_launch": avg_b, "unit": "GB/s", "achieved": ach,
         "traffic": traffic["dram_bytes"] if traffic else None,
         "hbm": {"peak": hbm, "peak_source": hbm_src, "model_frac": ach / hbm}}
    if traffic:
        r["hbm"]["dram_achieved"] = traffic["dram_bytes"] / screen_s / 1e9
        r["hbm"]["dram_frac"] = r["hbm"]["dram_achieved"] / hbm
        r["traffic_source"] = traffic["source"]
        r["traffic_launches"] = traffic.get("launches", 1)
    if ach > hbm and l2pk:
        # more algorithmic bytes per second than HBM can deliver: the postings
        # are mostly L2 hits, so the binding ceiling is the L2 read bandwidth
        r.update(bound="l2", peak=l2pk, peak_source=l2_src, frac=ach / l2pk)
    else:
        r.update(bound="hbm", peak=hbm, peak_source=hbm_src, frac=ach / hbm)
    if traffic and l2pk:
        la = traffic["l2_read_bytes"] / screen_s / 1e9
        r["l2"] = {"achieved": la, "peak": l2pk, "unit": "GB/s", "frac": la / l2pk,
                   "l2_read_bytes": traffic["l2_read_bytes"],
                   "what": "L2->SM bytes ncu counted for the launch (the layout's mask/offset "
                           "words and dense-span zeros included)"}
    return r


# ----------------------------------------------------------------- CPU baseline

def cpu_assign_kernel():
    """(callable, kind): the reference's own compiled kernel when oracle/_ref
    was built, else the C restatement."""
    from oracle import oracle as O

    ref = O.ref_kernels()
    if ref is not None:
        return ref.assign_ivf, "reference"
    return None, "port"


def cpu_assign(ip, terms, vals, inv, k, threads, labels=None):
    """Assign the rows of CSR `ip` (row offsets into terms/vals) on `threads`
    host threads (contiguous row shards).  Returns (labels, postings, seconds)."""
    import concurrent.futures as cf

    import numpy as np

    from oracle import oracle as O

    fn, _ = cpu_assign_kernel()
    n = ip.size - 1
    t0 = time.perf_counter()
    if fn is None:
        lab, _, _, post = O.assign_ivf(ip, terms, vals, inv[0], inv[1], inv[2], k, threads)
        return lab, post, time.perf_counter() - t0
    lab = np.empty(n, np.int32) if labels is None else labels
    bounds = [n * w // threads for w in range(threads + 1)]

    def work(w):
        lo, hi = bounds[w], bounds[w + 1]
        if hi <= lo:
            return 0
        rho = np.zeros(k)
        ctr = np.zeros(5, np.int64)
        fn(np.ascontiguousarray(ip[lo:hi + 1]), terms, vals, inv[0], inv[1], inv[2], rho,
           lab[lo:hi], ctr)
        return int(ctr[0])

    with cf.ThreadPoolExecutor(threads) as ex:
        post = sum(ex.map(work, range(threads)))
    return lab, post, time.perf_counter() - t0


def cpu_baseline_measure(ds, k, budget_s, labels, means):
    """The reference CPU path at the GPU run's state (its means and labels):
    the reference's own compiled kernel (oracle/_ref) on all host threads over
    a bounded row sample, scaled to N, plus the numpy update
    (variants.py:254-307) and the dense objective (clustering.py:105-119) on
    the full corpus.  A projection of one iteration from a sample — the
    reference arm (--impl reference) measures whole iterations."""
    import numpy as np

    from oracle import oracle as O

    threads = O.host_threads()
    m = O.Means(means.k, means.dim, np.asarray(means.indptr), np.asarray(means.term_ids),
                np.asarray(means.values), np.asarray(means.retained))
    inv = O.inverted(m)
    ip = np.asarray(ds.indptr)
    probe = min(ds.n, max(threads * 4, 64))
    _, _, tp = cpu_assign(ip[: probe + 1], ds.term_ids, ds.values, inv, k, threads)
    rows = int(min(ds.n, max(probe, probe * budget_s / max(tp, 1e-6))))
    _, _, ta = cpu_assign(ip[: rows + 1], ds.term_ids, ds.values, inv, k, threads)
    t0 = time.perf_counter()
    O.update(ds, labels, m)
    t_upd = time.perf_counter() - t0
    t0 = time.perf_counter()
    O.objective(ds, labels, m)
    t_obj = time.perf_counter() - t0
    _, kind = cpu_assign_kernel()
    per = ta * ds.n / rows + t_upd + t_obj
    sample = (f"assign: rows 0..{rows} of {ds.n} on {threads} threads "
              f"({'reference _kernels.assign_ivf (oracle/_ref)' if kind == 'reference' else 'C oracle'})"
              f" {ta:.2f}s, scaled to N; means and labels = the GPU run's state; update (numpy "
              f"restatement of variants.py:254-307, 1 thread) {t_upd:.2f}s and objective "
              f"{t_obj:.2f}s on the full corpus; CPU {cpu_model()}")
    return {"value": 1.0 / per, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample}


# ----------------------------------------------------------------- arms

def reference_arm(args, rank, world):
    """The reference CPU implementation of the path, timed on this host.

    Configs 0-1: real Lloyd iterations over the whole corpus (the reference's
    loop body, clustering.py:262-298): MeanSet.inverted (means.py:169-179),
    the reference's own compiled _kernels.assign_ivf on all host threads over
    contiguous row shards, objective_cosine's dense gather + fsum
    (clustering.py:105-119) and update_means (variants.py:254-307), from the
    same initial means (init_means, clustering.py:82-102) and warm-up count
    as our arm.  Configs 2-4 (a whole iteration takes minutes on the CPU):
    each step assigns a fixed seeded row sample and takes the objective over
    it; value = (sample fraction) / step time.  The corpus comes from the
    standalone generator (tools/_build/libcorpus.so): this process never maps
    libivfkm.so."""
    if rank != 0:
        return
    import numpy as np

    from oracle import oracle as O
    from paper_2002_09094_b200 import synth

    c, spec = workload(args.config)
    ds = synth.make_dataset(spec, standalone=True)
    k, threads = c["k"], O.host_threads()
    _, kind = cpu_assign_kernel()
    m = O.init_means(ds, k, c["seed"])
    full = args.config <= 1
    ip, terms, vals = np.asarray(ds.indptr), np.asarray(ds.term_ids), np.asarray(ds.values)
    frac = 1.0
    if not full:
        rng = np.random.default_rng(1234)
        ip0 = np.asarray(ds.indptr)
        rows = np.sort(rng.choice(ds.n, max(1, ds.n // 200), replace=False))
        lens = np.diff(ip0)[rows]
        ip = np.zeros(rows.size + 1, np.int64)
        np.cumsum(lens, out=ip[1:])
        idx = np.repeat(ip0[rows] - ip[:-1], lens) + np.arange(int(ip[-1]))
        terms, vals = terms[idx], vals[idx]
        frac = rows.size / ds.n

        class _Sub:
            indptr, term_ids, values, dim, n = ip, terms, vals, ds.dim, rows.size
        sub = _Sub
    parts = {"inverted": [], "assign": [], "objective": [], "update": []}
    steps = []
    prev = None
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        inv = O.inverted(m)  # MeanSet.inverted, built lazily by the next assign
        t1 = time.perf_counter()
        labels, post, _ = cpu_assign(ip, terms, vals, inv, k, threads)
        t2 = time.perf_counter()
        obj = O.objective(ds if full else sub, labels, m)
        t3 = time.perf_counter()
        if full:
            _ = prev is not None and np.array_equal(labels, prev)  # clustering.py:286
            m = O.update(ds, labels, m)
            prev = labels
        t4 = time.perf_counter()
        steps.append(t4 - t0)
        if i >= args.warmup:
            for key, dt in zip(parts, (t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
                parts[key].append(dt)
    timed = steps[args.warmup:]
    t = sum(timed)
    value = frac * len(timed) / t
    what = ("whole-corpus Lloyd iterations" if full else
            f"assign + objective of a fixed {frac:.4f} row sample per step at the initial means "
            "(value = sample fraction / step time)")
    sample = (f"{what}: reference _kernels.assign_ivf "
              f"({'oracle/_ref, compiled from the reference' if kind == 'reference' else 'C restatement'})"
              f" on {threads} threads, numpy update/objective restatements (1 thread); "
              f"per step s: " + ", ".join(f"{k_} {statistics.mean(v):.3f}" for k_, v in parts.items()
                                          if v) + f"; CPU {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * t / len(timed),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(args.config, c, spec, ds, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "cpu": {"model": cpu_model(), "threads": threads},
        "iteration_fraction_per_step": frac,
        "last_postings": int(post), "last_objective": obj,
    }
    print(json.dumps(line), flush=True)


def _engine_run(cfg, warmup, steps, world=1, events=True):
    """Build the config, run `warmup` + `steps` iterations on cuda:0; returns
    the measurements and the live state."""
    import torch

    from paper_2002_09094_b200 import synth
    from paper_2002_09094_b200.clustering import init_means
    from paper_2002_09094_b200.engine import DeviceDataset, HostDataset, LloydEngine

    dev = torch.device("cuda", 0)
    c, spec = workload(cfg)
    t_gen = time.perf_counter()
    ds = synth.make_dataset(spec)
    t_gen = time.perf_counter() - t_gen
    k = c["k"]
    means0 = init_means(ds, k, c["seed"], representation="sparse_inverted")
    hd = HostDataset(ds, pin=True, compact=True)  # 16-bit term gaps over PCIe
    dd = DeviceDataset(hd, dev)
    eng = LloydEngine(dd, k)
    dm = eng.upload_means(means0)
    torch.cuda.synchronize()
    prev = None
    for _ in range(warmup):
        lab = eng.assign(dm, prev)
        eng.read_stats()
        dm = eng.update(lab, dm)
        prev = lab
    torch.cuda.synchronize()
    out = {"ds": ds, "hd": hd, "dd": dd, "eng": eng, "c": c, "spec": spec, "k": k,
           "t_gen": t_gen}
    if steps == 0:
        out.update(dm=dm, prev=prev)
        return out
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    posts, changed, near = [], [], []
    launches0 = eng.launches
    clk = Clocks(0)
    torch.cuda.synchronize()
    start.record()
    for i in range(steps):
        evs[i][0].record()
        lab = eng.assign(dm, prev, events=ev[i])
        evs[i][1].record()
        eng.stats_async()  # read once the update has synchronised
        dm = eng.update(lab, dm)
        st = eng.stats_ready()
        posts.append(st.postings)
        changed.append(st.changed)
        near.append(st.near_ties)
        prev = lab
    end.record()
    torch.cuda.synchronize()
    clocks = clk.stop()
    total_ms = start.elapsed_time(end)
    screen_ms = [a.elapsed_time(b) for a, b in ev]
    assign_ms = [a.elapsed_time(b) for a, b in evs]
    n = ds.n
    bytes_alg = [algorithmic_bytes(p, ds.sum_nnz, n, eng.screen_bits // 8) for p in posts]
    out.update(dm=dm, prev=prev, lab=lab, clocks=clocks, total_ms=total_ms,
               screen_ms=screen_ms, assign_ms=assign_ms, posts=posts, changed=changed,
               near=near, launches=eng.launches - launches0,
               avg_b=sum(bytes_alg) / len(bytes_alg),
               avg_screen_s=sum(screen_ms) / len(screen_ms) / 1000.0)
    return out


def probe_arm(args):
    """Child of traffic_probe (under ncu): replay the run to its first timed
    screen launch."""
    import torch

    r = _engine_run(args.config, args.warmup, 0)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("probe")
    r["eng"].assign(r["dm"], r["prev"])
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()


def ours_arm(args, rank, world):
    import numpy as np
    import torch

    if world > 1 or args.dist:
        from paper_2002_09094_b200 import dist as D

        return D.bench_multi(args, rank, world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    r = _engine_run(args.config, args.warmup, args.steps)
    ds, hd, eng, c, spec, k = r["ds"], r["hd"], r["eng"], r["c"], r["spec"], r["k"]
    value = args.steps / (r["total_ms"] / 1000.0)
    screen_bits = eng.screen_bits

    # ---- end to end through host buffers
    from paper_2002_09094_b200.engine import HostIteration, StreamIteration

    e2e_steps = args.e2e_steps if args.e2e_steps is not None else max(3, min(args.steps, 10))
    host_means = r["dm"].to_meanset()
    last_labels = (r["lab"].cpu().numpy() + 1).astype(np.int32)
    del eng, r["eng"], r["dd"], r["dm"], r["lab"], r["prev"]
    torch.cuda.empty_cache()
    e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
           "steps": e2e_steps}
    if e2e_steps > 0:
        # (1) the corpus streamed in every step, labels + objective + counters
        # back; the means stay on the device (the model state, as in run())
        stream = StreamIteration(hd, k, host_means, dev)
        for _ in range(2):
            stream.step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            stream.step()
        torch.cuda.synchronize()
        e2e.update(value=e2e_steps / (time.perf_counter() - t0),
                   h2d_bytes_per_step=int(stream.last_h2d), d2h_bytes_per_step=int(stream.last_d2h),
                   what="corpus host->device every step (pinned), labels + objective + counters "
                        "device->host; means device-resident")
        del stream
        torch.cuda.empty_cache()
        # (2) stricter: the means also round-trip through host memory every step
        stepper = HostIteration(hd, k, dev)
        rt_steps = max(1, min(e2e_steps, 5))
        for _ in range(2):  # warm-up: both halves of the pinned double buffer
            _, host_means, _ = stepper.step(host_means)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(rt_steps):
            _, host_means, _ = stepper.step(host_means)
        torch.cuda.synchronize()
        e2e["means_roundtrip"] = {"value": rt_steps / (time.perf_counter() - t0),
                                  "h2d_bytes_per_step": int(stepper.last_h2d),
                                  "d2h_bytes_per_step": int(stepper.last_d2h)}
        del stepper
        torch.cuda.empty_cache()
        # (3) the public API: run("IVF", ds, k, seed, max_iter) on a host Dataset
        # (fresh Dataset object: its device copy is made inside the timed call)
        import paper_2002_09094_b200 as P

        ds2 = P.Dataset(ds.dim, ds.indptr, ds.term_ids, ds.values, normalized=True)
        iters = c["iters"]  # the config's own run length (BASELINE.json: 50 at config 1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = P.run("IVF", ds2, k, seed=c["seed"], max_iter=iters)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        e2e["run_api"] = {
            "value": res.iterations / dt, "unit": UNIT, "iterations": res.iterations,
            "seconds": dt, "h2d_bytes": int(ds.indptr.nbytes + ds.term_ids.nbytes
                                            + ds.values.nbytes),
            "d2h_bytes_per_step": int(ds.n * 4),
            "max_iter": iters, "converged": res.converged,
            "what": "paper_2002_09094_b200.run('IVF', ds, k, seed, max_iter) from a host "
                    "Dataset: corpus upload, init_means, BIVF builds, every iteration's labels "
                    "read back and digested into its IterationRecord, final means read back"}
        del res, ds2
        from paper_2002_09094_b200 import variants

        variants._ENGINES.clear()
        torch.cuda.empty_cache()

    traffic, traffic_note = None, None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r["total_ms"] / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "screen": f"fp{screen_bits} values, fp32 FMA, rigorous window -> exact f64 rescoring",
        "data": "synthetic", "config": config_dict(args.config, c, spec, ds, world),
        "postings_per_sec": sum(r["posts"]) / (sum(r["assign_ms"]) / 1000.0),
        "screen_postings_per_sec": sum(r["posts"]) / (sum(r["screen_ms"]) / 1000.0),
        "assign_ms": sum(r["assign_ms"]) / len(r["assign_ms"]),
        "screen_ms": sum(r["screen_ms"]) / len(r["screen_ms"]),
        "postings_per_step": sum(r["posts"]) // len(r["posts"]),
        "near_ties_per_step": sum(r["near"]) / len(r["near"]),
        "changed_per_step": sum(r["changed"]) / len(r["changed"]),
        "roofline": None, "e2e": e2e, "gpu_launches": r["launches"], "clocks": r["clocks"],
        "gen_seconds": r["t_gen"], "cpu": {"model": cpu_model()}, "csrc": csrc_digest(),
    }
    avg_b, avg_screen_s = r["avg_b"], r["avg_screen_s"]
    if not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline_measure(ds, k, args.cpu_seconds, last_labels,
                                                        host_means)
        except Exception as exc:  # the baseline must not sink the GPU number
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "port",
                                    "sample": f"failed: {exc!r}"}
    del r, hd, host_means
    torch.cuda.empty_cache()

    # ---- secondary: config 3 (largest single-GPU config) in the same run
    if not args.no_secondary and args.secondary_config != args.config:
        try:
            sc = args.secondary_config
            s = _engine_run(sc, 3, max(2, min(args.steps, 5)))
            sv = len(s["screen_ms"]) / (s["total_ms"] / 1000.0)
            line["secondary"] = {
                "config": config_dict(sc, s["c"], s["spec"], s["ds"], world), "value": sv,
                "unit": UNIT, "steps": len(s["screen_ms"]), "warmup": 3,
                "ms_per_step": s["total_ms"] / len(s["screen_ms"]),
                "screen_ms": s["avg_screen_s"] * 1000.0,
                "postings_per_step": sum(s["posts"]) // len(s["posts"]),
                "near_ties_per_step": sum(s["near"]) / len(s["near"]),
                "roofline": roofline(s["avg_b"], s["avg_screen_s"], stamped_traffic(sc),
                                     s["eng"].screen_bits),
                "clocks": s["clocks"], "gen_seconds": s["t_gen"]}
            del s
        except Exception as exc:
            line["secondary"] = {"error": repr(exc)}
        torch.cuda.empty_cache()

    if not args.no_traffic:
        traffic, traffic_note = traffic_probe(args.config, args.warmup)
    if traffic is None:
        traffic = stamped_traffic(args.config)
    line["roofline"] = roofline(avg_b, avg_screen_s, traffic, screen_bits)
    if traffic_note:
        line["roofline"]["traffic_note"] = traffic_note
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.probe:
        return probe_arm(args)
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    return ours_arm(args, rank, world)


if __name__ == "__main__":
    main()
