"""One steady-state Lloyd iteration inside an NVTX range "iter" (after
--warmup iterations), for per-kernel ncu launch lists of a single iteration:

    ncu --nvtx --nvtx-include "iter/" --metrics gpu__time_duration.sum --csv \\
        python tools/prof_iter.py --config 1
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2002_09094_b200 import synth  # noqa: E402
from paper_2002_09094_b200.clustering import init_means  # noqa: E402
from paper_2002_09094_b200.engine import DeviceDataset, HostDataset, LloydEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=6)
    a = ap.parse_args()
    c = synth.CONFIGS[a.config]
    ds = synth.make_dataset(c["corpus"])
    eng = LloydEngine(DeviceDataset(HostDataset(ds), "cuda"), c["k"])
    dm = eng.upload_means(init_means(ds, c["k"], c["seed"], "sparse_inverted"))
    prev = None
    for _ in range(a.warmup):
        lab = eng.assign(dm, prev)
        eng.read_stats()
        dm = eng.update(lab, dm)
        prev = lab
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("iter")
    lab = eng.assign(dm, prev)
    st = eng.read_stats()
    dm = eng.update(lab, dm)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print("changed", st.changed, "near_ties", st.near_ties)


if __name__ == "__main__":
    main()
