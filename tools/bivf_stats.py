"""Where the screen's work goes at a config: (object entry, span) pairs and
postings in the dense-prefix path vs the masked path, weighted by how many
objects hold each term (GPU tool)."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2002_09094_b200 import synth  # noqa: E402
from paper_2002_09094_b200.clustering import init_means  # noqa: E402
from paper_2002_09094_b200.engine import DeviceDataset, HostDataset, LloydEngine  # noqa: E402


def popc(x):
    x = x.to(torch.int64) & 0xFFFFFFFF
    x = x - ((x >> 1) & 0x55555555)
    x = (x & 0x33333333) + ((x >> 2) & 0x33333333)
    x = (x + (x >> 4)) & 0x0F0F0F0F
    return ((x * 0x01010101) & 0xFFFFFFFF) >> 24


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--iters", type=int, default=2)
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
    D, k, nblk = ds.dim, c["k"], eng.nblk
    h = dm.headers
    nh = D * nblk
    masks = h[:nh].view(D, nblk)
    offs = h[nh:2 * nh].view(D, nblk)
    nc = h[2 * nh + 1:2 * nh + 1 + D].to(torch.int64)
    dpre = h[2 * nh + 1 + D + 2 * k:2 * nh + 1 + D + 2 * k + D].to(torch.int64)
    ns = nblk // 8
    cnt = popc(masks).view(D, ns, 8).sum(2)                       # postings per (t, span)
    dense = ((offs.to(torch.int64) & 0x80000000) != 0).view(D, ns, 8)[:, :, 0]
    sidx = torch.arange(ns, device=h.device).view(1, ns)
    inpre = sidx < dpre.view(D, 1)
    no = torch.bincount(torch.from_numpy(np.asarray(ds.term_ids, np.int64) - 1).cuda(),
                        minlength=D).to(torch.float64)
    w = no.view(D, 1)
    out = {
        "config": a.config, "k": k, "spans": ns, "D": D,
        "pairs_prefix": float((w * inpre).sum()),
        "pairs_masked": float((w * (~inpre)).sum()),
        "pairs_masked_nonempty": float((w * ((~inpre) & (cnt > 0))).sum()),
        "pairs_masked_dense": float((w * ((~inpre) & dense)).sum()),
        "postings_prefix": float((w * cnt * inpre).sum()),
        "postings_masked": float((w * cnt * (~inpre)).sum()),
        "postings_masked_in_sparse_spans": float((w * cnt * ((~inpre) & ~dense)).sum()),
        "V": float((no * nc.to(torch.float64)).sum()),
        "screen_values": int(h[2 * nh].item()),
        "terms_with_prefix": int((dpre > 0).sum().item()),
        "sum_nc": int(nc.sum().item()),
        "sum_nc_in_prefix": int((cnt * inpre).sum().item()),
    }
    # object blocking potential: dense-prefix bytes a tile of B consecutive
    # objects (the screen's longest-first order) reads if each distinct term's
    # spans are fetched once per tile, against once per object
    terms = eng.dd.terms.long()
    rows = torch.repeat_interleave(torch.arange(ds.n, device=terms.device),
                                   eng.dd.row_ptr[1:] - eng.dd.row_ptr[:-1])
    rank = torch.empty(ds.n, dtype=torch.int64, device=terms.device)
    rank[eng.order.long()] = torch.arange(ds.n, device=terms.device)
    single = float(dpre[terms].sum())
    tiles = {}
    for B in (2, 4, 8, 16):
        key = torch.unique((rank[rows] // B) * D + terms)
        tiles[B] = float(dpre[key % D].sum()) / max(single, 1.0)
    out["dense_span_reads_tiled_fraction"] = tiles
    # dense-span reads (prefix + dense spans beyond it) by fill: share of the
    # (object entry, span) reads whose span holds (10 d)%..(10 d + 10)% of its
    # 256 slots — what a cheaper mid-fill representation could save
    dn = dense | inpre
    dec = torch.clamp((cnt * 10) // 256, max=9)
    wd = (w * dn).flatten()
    by = torch.zeros(10, dtype=torch.float64, device=h.device).index_add_(0, dec.flatten(), wd)
    out["dense_reads_by_fill_decile"] = (by / by.sum()).tolist()
    out["dense_reads_mean_fill"] = float((w * dn * cnt).sum() / (256.0 * (w * dn).sum()))
    hist = torch.bincount(cnt[~inpre & (cnt > 0)].flatten(), minlength=257)[:40].tolist()
    out["masked_nonempty_span_fill_hist"] = hist
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
