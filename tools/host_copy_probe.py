"""Host<->device copy paths for the public API's corpus upload and final
means read-back (GPU tool): pageable copies, the chunked pinned staging of
engine._upload with one or several host threads filling the stages, and the
reverse for device->host."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2002_09094_b200 import engine as E  # noqa: E402


def t(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return round(best * 1e3, 2)


def main():
    n = 69_000_000
    rng = np.random.default_rng(0)
    a64 = rng.random(n)
    a32 = rng.integers(0, 100000, n).astype(np.int32)
    res = {}
    dev = torch.device("cuda")
    res["pageable_h2d_f64"] = t(lambda: torch.from_numpy(a64).to(dev))
    for th in (1, 4, 8, 16):
        E.UPLOAD_THREADS = th
        res[f"staged_h2d_f64_{th}thr"] = t(lambda: E._upload(a64, dev))
        res[f"staged_h2d_i32_{th}thr"] = t(lambda: E._upload(a32, dev))
    d = torch.from_numpy(a64[:30_000_000]).to(dev)
    res["pageable_d2h_f64_240MB"] = t(lambda: d.cpu())
    for th in (1, 8):
        E.UPLOAD_THREADS = th
        res[f"staged_d2h_f64_240MB_{th}thr"] = t(lambda: E._download(d))
    res["pin_alloc_240MB+copy"] = t(lambda: d.to("cpu", non_blocking=False).pin_memory())
    print(res, flush=True)


if __name__ == "__main__":
    main()
