"""Sweep the fp32 screen kernel's tuning knobs on one config (GPU).

    python tools/sweep_screen.py --config 1 [--iters 2]

Builds realistic means (after --iters Lloyd iterations), then times
ivfkm_assign_screen for each (rr, rowcap) with CUDA events and prints
postings/s and ms per launch.  Results are checked against the default
plan's labels so a faster variant cannot be a wrong one.
"""

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
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--rr", default="0,8", help="0 = TMA screen, 2/4/8 = LDG screen, "
                    "-16*w = TMA screen with w warps per CTA")
    ap.add_argument("--rowcap", default="256,512,1024")
    ap.add_argument("--fill", default="0.5", help="BIVF dense_fill values (>1: never dense)")
    ap.add_argument("--permute", default="1")
    ap.add_argument("--smem", default="0", help="shared-memory budgets per CTA (0 = default)")
    ap.add_argument("--order", default="none", help="none,label: object processing order")
    ap.add_argument("--bits", type=int, default=16, help="screen value precision (16 or 32)")
    args = ap.parse_args()
    c = synth.CONFIGS[args.config]
    ds = synth.make_dataset(c["corpus"])
    eng = LloydEngine(DeviceDataset(HostDataset(ds), "cuda"), c["k"], screen_bits=args.bits)
    dm = eng.upload_means(init_means(ds, c["k"], c["seed"], "sparse_inverted"))
    prev = None
    for _ in range(args.iters):
        lab = eng.assign(dm, prev)
        eng.read_stats()
        dm = eng.update(lab, dm)
        prev = lab
    base = eng.assign(dm, None).clone()
    st = eng.read_stats()
    out = []
    import itertools
    last_bivf = None
    import ctypes
    orders = {"none": None, "label": torch.argsort(base.long(), stable=True).to(torch.int32),
              "rowlen": torch.argsort(-(eng.dd.row_ptr[1:] - eng.dd.row_ptr[:-1]),
                                      stable=True).to(torch.int32)}
    # cache-locality experiments: group objects by one of their terms (by
    # document frequency rank within the row: rarest / median / q-quantile)
    import numpy as np

    ip = np.asarray(ds.indptr)
    tt = np.asarray(ds.term_ids) - 1
    df = np.bincount(tt, minlength=ds.dim)
    lens = np.diff(ip)
    row = np.repeat(np.arange(ds.n), lens)
    key = df[tt].astype(np.int64) * (ds.dim + 1) + tt  # (df, term) per entry
    srt = np.lexsort((key, row))  # rows in order, entries by ascending df
    for name, q in (("mindf", 0.0), ("q25df", 0.25), ("meddf", 0.5)):
        pick = ip[:-1] + np.minimum((lens * q).astype(np.int64), np.maximum(lens - 1, 0))
        term = tt[srt[pick]]
        o = np.lexsort((np.arange(ds.n), term)).astype(np.int32)
        orders[name] = torch.from_numpy(o).to(eng.device)
    for oname in args.order.split(","):
      o = orders[oname]
      eng.order = o
      for fill, perm, smem, rr, rowcap in itertools.product(map(float, args.fill.split(",")),
                                                          map(int, args.permute.split(",")),
                                                          map(int, args.smem.split(",")),
                                                          map(int, args.rr.split(",")),
                                                          map(int, args.rowcap.split(","))):
        if True:
            if last_bivf != (fill, perm):
                eng.lib.ivfkm_set_bivf_options(fill, perm)
                eng.build_bivf(dm)
                last_bivf = (fill, perm)
            eng.lib.ivfkm_set_tuning(rowcap, smem if smem else -1, rr)
            eng.rowcap = rowcap
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            times = []
            for _ in range(args.reps):
                lab = eng.assign(dm, None, events=ev)
                torch.cuda.synchronize()
                times.append(ev[0].elapsed_time(ev[1]))
            ok = bool(torch.equal(lab, base))
            st2 = eng.read_stats()
            ms = min(times)
            rec = {"bits": args.bits, "order": oname, "fill": fill, "permute": perm, "smem": smem, "rr": rr, "rowcap": rowcap, "screen_ms": ms,
                   "postings_per_s": st.postings / (ms / 1e3), "labels_ok": ok,
                   "near_ties": st2.near_ties, "overflow": st2.overflow}
            out.append(rec)
            print(json.dumps(rec), flush=True)
    eng.lib.ivfkm_set_tuning(1024, 0, 0)
    eng.lib.ivfkm_set_tuning(1024, 0, -128)
    eng.lib.ivfkm_set_bivf_options(1.0 / 64.0, 1)  # the default


if __name__ == "__main__":
    main()
