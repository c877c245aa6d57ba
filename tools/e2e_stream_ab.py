"""A/B of the streamed end-to-end step (StreamIteration) with plain int32
term ids vs the compact 16-bit gaps (GPU box).

    python tools/e2e_stream_ab.py [config]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2002_09094_b200 import synth  # noqa: E402
from paper_2002_09094_b200.clustering import init_means  # noqa: E402
from paper_2002_09094_b200.engine import HostDataset, StreamIteration  # noqa: E402


def main():
    c = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
    ds = synth.make_dataset(c["corpus"])
    ms = init_means(ds, c["k"], c["seed"], "sparse_inverted")
    for compact in (False, True, False, True):
        hd = HostDataset(ds, pin=True, compact=compact)
        it = StreamIteration(hd, c["k"], ms, "cuda")
        for _ in range(14):  # past the early iterations' churn
            it.step()
        torch.cuda.synchronize()
        ts = []
        for _ in range(6):
            t = time.perf_counter()
            it.step()
            ts.append(time.perf_counter() - t)
        print(f"compact={compact} bytes={hd.nbytes} step ms: " +
              " ".join(f"{1e3 * x:.1f}" for x in ts), flush=True)
        del it, hd


if __name__ == "__main__":
    main()
