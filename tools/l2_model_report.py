"""The reference's LLC model, re-parameterised for the B200 L2 and the BIVF
(paper_2002_09094_b200/l2model.py), against the ncu-measured DRAM bytes of
the screen launch (GPU box):

    python tools/l2_model_report.py [config ...]

Builds the config's data, runs the bench's warm-up iterations (the
measurement point of profiles/traffic.json and the ncu captures), reads the
BIVF headers back, and prints z*, the modelled DRAM bytes per screen launch
for several usable-L2 fractions, and the measured value.
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2002_09094_b200 import l2model, synth  # noqa: E402
from paper_2002_09094_b200.clustering import init_means  # noqa: E402
from paper_2002_09094_b200.engine import DeviceDataset, HostDataset, LloydEngine  # noqa: E402

# measured DRAM bytes of the screen launch: profiles/traffic.json (ncu, the
# launch after the 3 warm-up iterations — the point modelled here)
MEASURED = {}


def main():
    cfgs = [int(a) for a in sys.argv[1:]] or [1, 2]
    tr = json.loads((Path(bench.ROOT) / "profiles" / "traffic.json").read_text())
    for ci in cfgs:
        c, spec = bench.workload(ci)
        ds = synth.make_dataset(spec)
        eng = LloydEngine(DeviceDataset(HostDataset(ds, pin=False), "cuda"), c["k"])
        dm = eng.upload_means(init_means(ds, c["k"], c["seed"], "sparse_inverted"))
        prev = None
        for _ in range(3):
            lab = eng.assign(dm, prev)
            eng.read_stats()
            dm = eng.update(lab, dm)
            prev = lab
        torch.cuda.synchronize()
        h = dm.headers.cpu().numpy()
        blocks = l2model.term_sectors(h, c["k"], ds.dim, eng.nblk)
        no = np.bincount(np.asarray(ds.term_ids, np.int64) - 1, minlength=ds.dim)
        meas = (tr.get(f"config{ci}", {}) or {}).get("dram_bytes") or MEASURED.get(ci)
        for u in (0.5, 0.75, 0.9):
            r = l2model.predict_dram_bytes(no, blocks, ds.n, l2model.CacheParams(usable=u))
            print(json.dumps({"config": ci, "usable_l2": u, "z_star": r["z_star"],
                              "reachable_GB": round(r["reachable_bytes"] / 1e9, 3),
                              "blocks_per_scan": round(r["blocks_per_scan"]),
                              "model_dram_GB": round(r["dram_bytes"] / 1e9, 2),
                              "ncu_dram_GB": round(meas / 1e9, 2) if meas else None}),
                  flush=True)
        del eng, dm, lab, prev
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
