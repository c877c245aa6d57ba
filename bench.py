#!/usr/bin/env python
"""Benchmark of the B200 IVF spherical k-means Lloyd path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A *step* is one Lloyd iteration over the whole (synthetic) corpus: assign
(fp32 register screen + exact fp64 rescoring, changed-label count, sizes,
exact objective), the host-side convergence read, and the update (bit-exact
means + bitmap-block inverted-file rebuild).  Default workload is
BASELINE.json configs[1] (N=300k, D=100k, k=1000); ``--config 0..4`` picks
another.  Prints ONE JSON line (rank 0).

``value``  = Lloyd iterations/s with the corpus resident in HBM (CUDA events
             on the launching stream, barrier + synchronize on both sides, max
             over ranks);
``e2e``    = the same metric through host buffers: every step copies the
             corpus host->device from pinned memory and reads the step's
             result (labels, objective, counters) back, the means staying on
             the device as the model state (``e2e.means_roundtrip``: the
             stricter variant that also moves the means both ways);
``roofline`` = the screen kernel (dominant) against measured HBM: the
             algorithmic bytes of an assign pass in this layout (SURVEY.md §8(d)
             with b_p = the screen's value bytes): b_p * V +
             20 B * sum_nnz + 8 B * (N+1) + 8 B * N, over its average launch time
             (CUDA events); ``roofline.l2`` sets the L2->SM bytes ncu measured
             for the kernel (profiles/traffic.json) against the measured L2
             read bandwidth (profiles/l2_peak.json);
``cpu_baseline`` = the reference's own compiled kernel (oracle/_ref, or the
             C oracle restatement when it was not built) on this host's cores,
             on a bounded row sample, plus the numpy update; test
             infrastructure used only as the baseline, never on our path.

``--impl reference`` times that CPU implementation as the reference arm.
"""

from __future__ import annotations

import argparse
import json
import os
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
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


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


def l2_model(cfg_index, screen_s):
    """roofline.l2: ncu's L2->SM read bytes per screen launch (profiles/
    traffic.json, same config) over the live launch time, against the L2 read
    bandwidth measured by tools/l2_peak.cu (profiles/l2_peak.json)."""
    try:
        tr = json.loads((ROOT / "profiles" / "traffic.json").read_text()).get(f"config{cfg_index}")
        pk = json.loads((ROOT / "profiles" / "l2_peak.json").read_text())
        peak = max(r["GB_per_s"] for r in pk["results"] if r["buffer_mb"] * 2**20 < pk["l2_bytes"])
    except Exception:
        return None
    if not isinstance(tr, dict) or not tr.get("l2_read_bytes"):
        return None
    ach = tr["l2_read_bytes"] / screen_s / 1e9
    return {"achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "l2_read_bytes": tr["l2_read_bytes"], "source": "ncu lts__t_sectors_srcunit_tex_op_read"}


# ----------------------------------------------------------------- CPU baseline

def cpu_assign_kernel():
    """(callable, kind): the reference's own compiled kernel when oracle/_ref
    was built, else the C restatement."""
    from oracle import oracle as O

    ref = O.ref_kernels()
    if ref is not None:
        return ref.assign_ivf, "reference"
    return None, "port"


def cpu_sample_assign(ds, inv, k, rows, threads):
    """Assign rows [0, rows) with `threads` threads; returns seconds."""
    import concurrent.futures as cf

    import numpy as np

    from oracle import oracle as O

    fn, kind = cpu_assign_kernel()
    ip = np.ascontiguousarray(ds.indptr[: rows + 1])
    t0 = time.perf_counter()
    if fn is None:
        O.assign_ivf(ip, ds.term_ids, ds.values, inv[0], inv[1], inv[2], k, threads)
    else:
        bounds = [rows * w // threads for w in range(threads + 1)]

        def work(w):
            lo, hi = bounds[w], bounds[w + 1]
            if hi <= lo:
                return 0
            rho = np.zeros(k)
            lab = np.empty(hi - lo, np.int32)
            ctr = np.zeros(5, np.int64)
            fn(np.ascontiguousarray(ds.indptr[lo:hi + 1]), ds.term_ids, ds.values,
               inv[0], inv[1], inv[2], rho, lab, ctr)
            return int(ctr[0])

        with cf.ThreadPoolExecutor(threads) as ex:
            list(ex.map(work, range(threads)))
    return time.perf_counter() - t0


def cpu_baseline_measure(ds, k, seed, budget_s, steps=1, labels=None, means=None):
    """Time the reference CPU path on this host: all-core sampled assign with
    the reference's own compiled kernel (oracle/_ref; the C restatement when
    it was not built), extrapolated to N, plus the numpy update
    (variants.py:254-307) and objective on the full corpus.

    ``means``/``labels``: the state the GPU arm is timing (same iteration);
    without them the means are warmed by one update from seeded random labels
    (untimed) so the postings per object resemble a steady-state iteration
    rather than the sparse initial means."""
    import numpy as np

    from oracle import oracle as O

    threads = O.host_threads()
    rng = np.random.default_rng(0)
    if means is None:
        m0 = O.init_means(ds, k, seed)
        warm = rng.integers(1, k + 1, size=ds.n).astype(np.int32)
        m = O.update(ds, warm, m0)
    else:
        m = O.Means(means.k, means.dim, np.asarray(means.indptr), np.asarray(means.term_ids),
                    np.asarray(means.values), np.asarray(means.retained))
    if labels is None:
        labels = rng.integers(1, k + 1, size=ds.n).astype(np.int32)
    inv = O.inverted(m)
    probe = min(ds.n, max(threads * 4, 64))
    tp = cpu_sample_assign(ds, inv, k, probe, threads)
    rows = int(min(ds.n, max(probe, probe * budget_s / max(tp, 1e-6))))
    t0 = time.perf_counter()
    O.update(ds, labels, m)
    t_upd = time.perf_counter() - t0
    t0 = time.perf_counter()
    O.objective(ds, labels, m)
    t_obj = time.perf_counter() - t0
    per_step = []
    for _ in range(steps):
        ta = cpu_sample_assign(ds, inv, k, rows, threads) * ds.n / rows
        per_step.append(ta + t_upd + t_obj)
    _, kind = cpu_assign_kernel()
    sample = (f"assign: {rows} of {ds.n} rows on {threads} threads "
              f"({'reference _kernels.assign_ivf (oracle/_ref)' if kind == 'reference' else 'C oracle'}), "
              f"scaled to N, means {'= the GPU run state' if means is not None else 'warmed by one update'}; "
              f"update (numpy restatement of variants.py:254-307, 1 thread) {t_upd:.2f}s and "
              f"objective {t_obj:.2f}s on the full corpus")
    return {"threads": threads, "kind": kind, "sample": sample, "t_update": t_upd,
            "t_objective": t_obj}, per_step


# ----------------------------------------------------------------- arms

def reference_arm(args, rank, world):
    if rank != 0:
        return
    from paper_2002_09094_b200 import synth

    c, spec = workload(args.config)
    ds = synth.make_dataset(spec)
    info, per = cpu_baseline_measure(ds, c["k"], c["seed"], args.cpu_seconds,
                                     steps=args.steps + args.warmup)
    timed = per[args.warmup:]
    t = sum(timed)
    value = len(timed) / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * t / len(timed),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(args.config, c, spec, ds, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": info["threads"],
                         "kind": info["kind"], "sample": info["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def ours_arm(args, rank, world):
    import numpy as np
    import torch

    from paper_2002_09094_b200 import synth
    from paper_2002_09094_b200.clustering import init_means
    from paper_2002_09094_b200.engine import (DeviceDataset, DeviceMeans, HostDataset,
                                              LloydEngine)

    if world > 1 or args.dist:
        from paper_2002_09094_b200 import dist as D

        return D.bench_multi(args, rank, world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    c, spec = workload(args.config)
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
    for _ in range(args.warmup):
        lab = eng.assign(dm, prev)
        st = eng.read_stats()
        dm = eng.update(lab, dm)
        prev = lab
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    posts, changed, near = [], [], []
    launches0 = eng.launches
    clk = Clocks(0)
    torch.cuda.synchronize()
    start.record()
    for i in range(args.steps):
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
    launches = eng.launches - launches0
    total_ms = start.elapsed_time(end)
    screen_ms = [a.elapsed_time(b) for a, b in ev]
    assign_ms = [a.elapsed_time(b) for a, b in evs]
    value = args.steps / (total_ms / 1000.0)
    n = ds.n
    bytes_alg = [algorithmic_bytes(p, ds.sum_nnz, n, eng.screen_bits // 8) for p in posts]
    avg_b = sum(bytes_alg) / len(bytes_alg)
    avg_screen_s = sum(screen_ms) / len(screen_ms) / 1000.0
    achieved = avg_b / avg_screen_s / 1e9
    peak, peak_kind = measured_peak_hbm()
    traffic = None
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists():
        try:
            tr = json.loads(tp.read_text()).get(f"config{args.config}")
            traffic = tr.get("dram_bytes") if isinstance(tr, dict) else tr
        except Exception:
            traffic = None

    # ---- end to end through host buffers: every step uploads the corpus and the
    # current means from pinned memory and reads labels + new means back
    from paper_2002_09094_b200.engine import HostIteration, StreamIteration

    e2e_steps = args.e2e_steps if args.e2e_steps is not None else max(3, min(args.steps, 10))
    host_means = dm.to_meanset()
    last_labels = (lab.cpu().numpy() + 1).astype(np.int32)
    screen_bits = eng.screen_bits
    del eng, dd, dm, lab, prev  # the e2e engines below bring their own device state
    torch.cuda.empty_cache()
    h2d = d2h = 0
    e2e_value = e2e_rt = None
    rt_h2d = rt_d2h = 0
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
        e2e_value = e2e_steps / (time.perf_counter() - t0)
        h2d, d2h = stream.last_h2d, stream.last_d2h
        del stream
        torch.cuda.empty_cache()
        # (2) stricter: the means also round-trip through host memory every
        # step (the reference's assign/update API on host arrays)
        stepper = HostIteration(hd, k, dev)
        rt_steps = max(1, min(e2e_steps, 5))
        for _ in range(2):  # warm-up: both halves of the pinned double buffer
            _, host_means, _ = stepper.step(host_means)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(rt_steps):
            labels_e2e, host_means, _ = stepper.step(host_means)
        torch.cuda.synchronize()
        e2e_rt = rt_steps / (time.perf_counter() - t0)
        rt_h2d, rt_d2h = stepper.last_h2d, stepper.last_d2h
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "screen": f"fp{screen_bits} values, fp32 FMA, rigorous window -> exact f64 rescoring",
        "data": "synthetic", "config": config_dict(args.config, c, spec, ds, world),
        "postings_per_sec": sum(posts) / (sum(assign_ms) / 1000.0),
        "screen_postings_per_sec": sum(posts) / (sum(screen_ms) / 1000.0),
        "assign_ms": sum(assign_ms) / len(assign_ms),
        "screen_ms": sum(screen_ms) / len(screen_ms),
        "postings_per_step": sum(posts) // len(posts),
        "near_ties_per_step": sum(near) / len(near), "changed_per_step": sum(changed) / len(changed),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                     "kernel": f"screen_kernel (BIVF register screen, fp{screen_bits} values)",
                     "bytes_per_launch": avg_b, "l2": l2_model(args.config, avg_screen_s)},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
                "what": "corpus host->device every step (pinned), labels + objective + "
                        "counters device->host; means device-resident",
                "means_roundtrip": {"value": e2e_rt, "h2d_bytes_per_step": int(rt_h2d),
                                    "d2h_bytes_per_step": int(rt_d2h)}},
        "gpu_launches": launches,
        "clocks": clocks,
        "gen_seconds": t_gen,
    }
    if not args.no_cpu_baseline:
        try:
            info, per = cpu_baseline_measure(ds, k, c["seed"], args.cpu_seconds, steps=1,
                                             labels=last_labels, means=host_means)
            line["cpu_baseline"] = {"value": 1.0 / per[0], "unit": UNIT, "cores": info["threads"],
                                    "kind": info["kind"], "sample": info["sample"]}
        except Exception as exc:  # baseline must not sink the GPU number
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "port",
                                    "sample": f"failed: {exc!r}"}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    return ours_arm(args, rank, world)


if __name__ == "__main__":
    main()
