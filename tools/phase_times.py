"""Per-phase device time of a Lloyd iteration (CUDA events on the compute
stream): screen, finish (rescoring + sizes + objective), stats read, update
(count + fill), BIVF rebuild; plus the step total and the host gaps it
implies.  GPU tool."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2002_09094_b200 import synth  # noqa: E402
from paper_2002_09094_b200.clustering import init_means  # noqa: E402
from paper_2002_09094_b200 import engine as E  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--update-option", type=int, nargs=2, action="append", default=[],
                    metavar=("WHICH", "VALUE"), help="ivfkm_set_update_option before the run")
    a = ap.parse_args()
    from paper_2002_09094_b200 import _lib
    for w, v in a.update_option:
        _lib.check(_lib.load().ivfkm_set_update_option(w, v), "ivfkm_set_update_option")
    c = synth.CONFIGS[a.config]
    ds = synth.make_dataset(c["corpus"])
    eng = E.LloydEngine(E.DeviceDataset(E.HostDataset(ds), "cuda"), c["k"])
    dm = eng.upload_means(init_means(ds, c["k"], c["seed"], "sparse_inverted"))
    prev = None
    for _ in range(a.warmup):
        lab = eng.assign(dm, prev)
        eng.read_stats()
        dm = eng.update(lab, dm)
        prev = lab
    torch.cuda.synchronize()
    orig_build = eng.build_bivf
    marks = {}

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def build(dm_):
        marks["bivf0"] = ev()
        out = orig_build(dm_)
        marks["bivf1"] = ev()
        return out

    eng.build_bivf = build
    rows = []
    for _ in range(a.steps):
        t0 = ev()
        s = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        lab = eng.assign(dm, prev, events=s)
        t1 = ev()
        eng.stats_async()
        dm = eng.update(lab, dm)
        eng.stats_ready()
        t2 = ev()
        torch.cuda.synchronize()
        r = {"step": t0.elapsed_time(t2), "screen": s[0].elapsed_time(s[1]),
             "finish": s[1].elapsed_time(t1), "update": t1.elapsed_time(marks["bivf0"]),
             "bivf": marks["bivf0"].elapsed_time(marks["bivf1"]),
             "after_bivf": marks["bivf1"].elapsed_time(t2)}
        rows.append(r)
        prev = lab
    avg = {k: sum(r[k] for r in rows) / len(rows) for k in rows[0]}
    print(json.dumps({"config": a.config, "update_option": a.update_option, "ms": avg}),
          flush=True)


if __name__ == "__main__":
    main()
