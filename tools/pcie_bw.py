"""Host<->device copy bandwidth from pinned memory (context for the e2e number)."""
import json
import time

import torch


def main():
    n = 1 << 28  # 1 GiB of float32
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    out = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        out[name + "_GBps"] = 5 * 4 * n / (time.perf_counter() - t) / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
