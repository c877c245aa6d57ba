"""Break an e2e step (HostIteration) into host-visible phases (GPU box)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2002_09094_b200 import synth  # noqa: E402
from paper_2002_09094_b200.clustering import init_means  # noqa: E402
from paper_2002_09094_b200.engine import HostDataset, HostIteration  # noqa: E402


def main():
    c = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
    ds = synth.make_dataset(c["corpus"])
    hd = HostDataset(ds, pin=True)
    ms = init_means(ds, c["k"], c["seed"], "sparse_inverted")
    for prefetch in (True, False):
        it = HostIteration(hd, c["k"], "cuda", prefetch=prefetch)
        for _ in range(3):
            _, ms, _ = it.step(ms)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            t = time.perf_counter()
            _, ms, _ = it.step(ms)
            ts.append(time.perf_counter() - t)
        print(f"prefetch={prefetch} step ms: " + " ".join(f"{1e3 * x:.1f}" for x in ts))
    # phase timing without prefetch
    import cProfile
    import pstats

    it = HostIteration(hd, c["k"], "cuda", prefetch=True)
    _, ms, _ = it.step(ms)
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(3):
        _, ms, _ = it.step(ms)
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(18)


if __name__ == "__main__":
    main()
