"""The paper's IVF vs IVFD contrast on the B200: one assign of each at the
same means (steady state after --iters iterations), CUDA events, labels
compared (IVF argmax vs IVFD rule differ only where nothing beats 0.0)."""
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
    ap.add_argument("--iters", type=int, default=3)
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
    out = {"config": a.config}
    eng.objects_inverted()  # once per corpus, outside the timing
    for name, rule in (("ivf", 0), ("ivfd_native", 1)):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize()
        ev[0].record()
        lab = eng.assign(dm, None, rule=rule)
        ev[1].record()
        st = eng.read_stats()
        out[name] = {"assign_ms": ev[0].elapsed_time(ev[1]), "postings": st.postings,
                     "objective": st.objective}
        out[name + "_labels"] = lab.clone()
    same = int((out.pop("ivf_labels") == out.pop("ivfd_native_labels")).sum().item())
    out["labels_equal"] = same
    out["N"] = ds.n
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
