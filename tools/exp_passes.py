"""Experiment: the screen as slot-range passes (R launches over all objects,
each covering 1/R of the slots) against the one-pass plan.  Timing only —
labels of the pass mode are not final (no cross-pass merge)."""
import argparse
import json
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
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--passes", default="0,2,4,8,16")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--pf", default="0")
    ap.add_argument("--warps", default="0")
    ap.add_argument("--rowcap", default="0", help="0: the engine's")
    ap.add_argument("--maxreg", default="56", help="(recorded only)")
    ap.add_argument("--presort", default="1", help="pass mode stages presorted rows: 1,0")
    ap.add_argument("--tma", default="0", help="(removed variant)")
    ap.add_argument("--hot", default="0", help="(removed variant)")
    ap.add_argument("--fill", default="0.015625", help="BIVF dense_fill values to sweep")
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
    import itertools

    from bench import Clocks
    rc0 = eng.rowcap
    base = None
    last_fill = None
    for fill, r, pf, w, rc, mr, ps, tm, hot in itertools.product(map(float, a.fill.split(",")),map(int, a.passes.split(",")),
                                                      map(int, a.pf.split(",")),
                                                      map(int, a.warps.split(",")),
                                                      map(int, a.rowcap.split(",")),
                                                      map(int, a.maxreg.split(",")),
                                                      map(int, a.presort.split(",")),
                                                      map(int, a.tma.split(",")),
                                                      map(int, a.hot.split(","))):
        eng.presort = bool(ps)
        if fill != last_fill:
            eng.lib.ivfkm_set_bivf_options(fill, 1)
            dm = eng.build_bivf(dm)
            last_fill = fill
        eng.lib.ivfkm_set_screen_warps(w)
        eng.rowcap = rc or rc0
        eng.passes = r if r > 0 else None  # 0: the engine's plan
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ts = []
        clk = Clocks(0)
        for _ in range(a.reps):
            lab = eng.assign(dm, None, events=ev)
            torch.cuda.synchronize()
            ts.append(ev[0].elapsed_time(ev[1]))
        lab = lab.clone()
        if base is None:
            base = lab
        ok = bool(torch.equal(lab, base))
        st = eng.read_stats()
        ck = clk.stop() or {}
        print(json.dumps({"sm_mhz": ck.get("sm_mhz"), "reasons": ck.get("reasons"), "config": a.config, "passes": r, "planned": eng.screen_passes(dm), "warps": w, "rowcap": eng.rowcap,
                          "maxreg": mr, "presort": ps, "fill": fill, "labels_ok": ok, "screen_ms": min(ts), "all": ts,
                          "postings": st.postings}), flush=True)
    eng.lib.ivfkm_set_screen_warps(0)
    eng.lib.ivfkm_set_bivf_options(1.0 / 64.0, 1)


if __name__ == "__main__":
    main()
