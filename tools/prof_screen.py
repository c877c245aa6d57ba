"""Run a config to steady state and issue one more assign inside an NVTX
range "profile", for ncu captures of the screen at that state:

    ncu --nvtx --nvtx-include "profile/" -k regex:screen_kernel -c 1 --set full \\
        python tools/prof_screen.py --config 3
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
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--passes", type=int, default=0, help="0: the engine's plan")
    a = ap.parse_args()
    c = synth.CONFIGS[a.config]
    ds = synth.make_dataset(c["corpus"])
    eng = LloydEngine(DeviceDataset(HostDataset(ds), "cuda"), c["k"])
    dm = eng.upload_means(init_means(ds, c["k"], c["seed"], "sparse_inverted"))
    prev = None
    for _ in range(a.iters):
        lab = eng.assign(dm, prev)
        eng.read_stats()
        dm = eng.update(lab, dm)
        prev = lab
    eng.passes = a.passes or None
    print("passes", eng.screen_passes(dm), flush=True)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("profile")
    eng.assign(dm, prev)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
