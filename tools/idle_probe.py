"""Where does the device sit idle inside a Lloyd iteration?

    python tools/idle_probe.py [--config 1] [--steps 3]

Runs the bench's engine loop (warm-up first), records the timed iterations
with the torch profiler (CUPTI kernel and memcpy activity), and prints the
device-busy time, the wall span and the largest gaps between consecutive
device activities with their neighbours.  Diagnostic only (never a bench
number: the profiler adds its own overhead).
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import bench
    from paper_2002_09094_b200 import synth
    from paper_2002_09094_b200.clustering import init_means
    from paper_2002_09094_b200.engine import DeviceDataset, HostDataset, LloydEngine

    dev = torch.device("cuda", 0)
    c, spec = bench.workload(a.config)
    ds = synth.make_dataset(spec)
    means0 = init_means(ds, c["k"], c["seed"], representation="sparse_inverted")
    eng = LloydEngine(DeviceDataset(HostDataset(ds, pin=True), dev), c["k"])
    dm = eng.upload_means(means0)
    prev = None
    for _ in range(a.warmup):
        lab = eng.assign(dm, prev)
        eng.read_stats()
        dm = eng.update(lab, dm)
        prev = lab
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(a.steps):  # the bench's loop
            lab = eng.assign(dm, prev)
            eng.stats_async()
            dm = eng.update(lab, dm)
            eng.stats_ready()
            prev = lab
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in evs)
    if not iv:
        print("no device activity recorded")
        return
    busy, cur_s, cur_e = 0.0, iv[0][0], iv[0][1]
    gaps = []
    last_name = iv[0][2]
    for s, e, n in iv[1:]:
        if s > cur_e:
            busy += cur_e - cur_s
            gaps.append((s - cur_e, last_name[:60], n[:60]))
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
        last_name = n
    busy += cur_e - cur_s
    span = iv[-1][1] - iv[0][0]
    print(f"steps {a.steps}: span {span / 1e3:.3f} ms, device busy {busy / 1e3:.3f} ms, "
          f"idle {(span - busy) / 1e3:.3f} ms ({(span - busy) / a.steps / 1e3:.3f} ms per step)")
    gaps.sort(reverse=True)
    for g, before, after in gaps[:25]:
        print(f"  gap {g:8.1f} us  after {before}  before {after}")


if __name__ == "__main__":
    main()
