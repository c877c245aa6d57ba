"""Time the public API run("IVF", ds, k, seed, max_iter) at several run
lengths (fresh Dataset objects, so the device copy and the engine are made
inside each timed call, as in bench.py's e2e.run_api), and the time of each
iteration inside one run.  GPU tool."""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2002_09094_b200 as P  # noqa: E402
from paper_2002_09094_b200 import synth, variants  # noqa: E402
from paper_2002_09094_b200.engine import LloydEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--iters", type=int, nargs="+", default=[1, 5, 50])
    ap.add_argument("--profile", action="store_true")
    a = ap.parse_args()
    c = synth.CONFIGS[a.config]
    ds = synth.make_dataset(c["corpus"])
    out = {"config": a.config, "run_s": {}}
    for it in [1] + a.iters:  # the first call warms the allocator and the libraries
        d2 = P.Dataset(ds.dim, ds.indptr, ds.term_ids, ds.values, normalized=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.run("IVF", d2, c["k"], seed=c["seed"], max_iter=it)
        torch.cuda.synchronize()
        out["run_s"][it] = time.perf_counter() - t0
        del d2
        variants._ENGINES.clear()
        torch.cuda.empty_cache()
    if a.profile:
        import cProfile
        import io
        import pstats

        d2 = P.Dataset(ds.dim, ds.indptr, ds.term_ids, ds.values, normalized=True)
        pr = cProfile.Profile()
        torch.cuda.synchronize()
        pr.enable()
        P.run("IVF", d2, c["k"], seed=c["seed"], max_iter=5)
        torch.cuda.synchronize()
        pr.disable()
        buf = io.StringIO()
        pstats.Stats(pr, stream=buf).sort_stats("cumulative").print_stats(30)
        print(buf.getvalue(), flush=True)
        del d2
        variants._ENGINES.clear()
        torch.cuda.empty_cache()
    # the fixed cost of a run, phase by phase
    from paper_2002_09094_b200.clustering import init_means
    from paper_2002_09094_b200.engine import DeviceDataset

    ph = {}

    def mark(name, t0):
        torch.cuda.synchronize()
        t = time.perf_counter()
        ph[name] = round(1e3 * (t - t0), 2)
        return t

    d2 = P.Dataset(ds.dim, ds.indptr, ds.term_ids, ds.values, normalized=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    means = init_means(d2, c["k"], c["seed"], representation="sparse_inverted")
    t = mark("init_means", t)
    dd = DeviceDataset.from_dataset(d2, "cuda")
    t = mark("upload", t)
    eng = LloydEngine(dd, c["k"])
    t = mark("engine", t)
    dm = eng.upload_means(means)
    t = mark("upload_means", t)
    lab = eng.assign(dm, None)
    t = mark("assign1", t)
    eng.read_stats()
    lab.cpu()
    t = mark("read1", t)
    eng.update(lab, dm)
    t = mark("update1", t)
    out["fixed_ms"] = ph
    del eng, dd, d2
    torch.cuda.empty_cache()
    # per-iteration host time stamps inside one run (assign entry to assign entry)
    stamps = []
    orig = LloydEngine.assign

    def assign(self, *args, **kw):
        torch.cuda.synchronize()
        stamps.append(time.perf_counter())
        return orig(self, *args, **kw)

    LloydEngine.assign = assign
    d2 = P.Dataset(ds.dim, ds.indptr, ds.term_ids, ds.values, normalized=True)
    P.run("IVF", d2, c["k"], seed=c["seed"], max_iter=max(a.iters))
    LloydEngine.assign = orig
    out["iter_ms_synced"] = [round(1e3 * (b - a_), 2) for a_, b in zip(stamps, stamps[1:])]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
