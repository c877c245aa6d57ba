"""Generate the golden fixtures by running the REFERENCE itself.

Run here (the reference is mounted read-only at /root/reference; it does not
exist on the GPU box, so its outputs are committed as .npz fixtures):

    python tests/golden/make_golden.py

The reference `run("IVF", ...)` is executed through its own public API with
its compiled Cython kernel (oracle/_ref, built by oracle/build_ref.sh) and,
as a cross-check, its numpy backend.  Inputs come from the package's seeded
generator (paper_2002_09094_b200.synth); small cases store the inputs too,
config 0 stores a SHA-256 of the regenerated inputs instead.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import sparse_kmeans as sk  # noqa: E402  (the reference package)
from sparse_kmeans import kernels as skk  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2002_09094_b200 import synth  # noqa: E402

OUT = Path(__file__).resolve().parent

ref_k = O.ref_kernels()
if ref_k is None:
    raise SystemExit("build oracle/_ref first: oracle/build_ref.sh")
skk._MODULES["compiled"] = ref_k


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def run_ref(ds, k, seed, max_iter, backend="compiled", variant="IVF"):
    res = sk.run(variant, ds, k, seed=seed, max_iter=max_iter, backend=backend,
                 keep_history=True)
    return res


def dump(name, ds, k, seed, max_iter, store_inputs=True, extra=None, variant="IVF"):
    res = run_ref(ds, k, seed, max_iter, variant=variant)
    res_py = run_ref(ds, k, seed, max_iter, backend="python", variant=variant)
    assert [r.assignment_digest for r in res.records] == \
        [r.assignment_digest for r in res_py.records], "reference backends disagree"
    labels = np.stack([r.labels for r in res.records]).astype(np.int32)
    # top-two gaps under the means of each iteration (dense; small cases only)
    gaps = []
    for m in res.history_means:
        _, t1, t2, _ = O.assign_ivf(ds.indptr, ds.term_ids, ds.values,
                                    m.inverted.indptr, m.inverted.owner_ids,
                                    m.inverted.values, m.k)
        gaps.append(t1 - t2)
    fm = res.final_means
    payload = dict(
        variant=np.array(variant), k=k, seed=seed, max_iter=max_iter, dim=ds.dim,
        converged=res.converged, iterations=res.iterations,
        objectives=np.array(res.objectives, dtype=np.float64),
        digests=np.array([r.assignment_digest for r in res.records], dtype=np.uint64),
        mults=np.array([r.counters.mults for r in res.records], dtype=np.int64),
        volume_ivf=np.array([r.volume_ivf for r in res.records], dtype=np.int64),
        mean_terms_total=np.array([r.mean_terms_total for r in res.records], dtype=np.int64),
        labels=labels, min_gap=np.array([g.min() for g in gaps]),
        final_indptr=fm.indptr, final_terms=fm.term_ids, final_values=fm.values,
        final_retained=fm.retained, final_sizes=res.final_assignment.sizes,
        inputs_sha=sha(ds.indptr, ds.term_ids, ds.values),
        # the reference's own JSON record of the run (clustering.py:206-226),
        # minus the backend name, for a byte-level comparison
        run_json=np.array(json.dumps(_strip_backend(res.to_json_dict()), sort_keys=True)),
    )
    if store_inputs:
        payload.update(indptr=ds.indptr, term_ids=ds.term_ids, values=ds.values)
    else:  # large case: keep the fixture small, pin the final means by hash
        payload["final_sha"] = sha(fm.indptr, fm.term_ids, fm.values, fm.retained)
        for key in ("final_terms", "final_values"):
            payload.pop(key)
        payload["labels"] = labels.astype(np.int16)
    if extra:
        payload.update(extra)
    np.savez_compressed(OUT / f"{name}.npz", **payload)
    print(f"{name}: iters={res.iterations} converged={res.converged} "
          f"min_gap={min(g.min() for g in gaps):.3g} obj={res.objectives[-1]:.12g}")


def _strip_backend(d):
    d = dict(d)
    d["meta"] = {k: v for k, v in d["meta"].items() if k != "backend"}
    return d


def ref_dataset(indptr, terms, vals, dim):
    return sk.Dataset(dim, indptr, terms, vals, normalized=True)


def main(only_ivfd=False):
    # 1) small synthetic with the config-0 distributions, several k
    spec = synth.CONFIGS[0]["corpus"].scaled(2000, 500, seed=7)
    ip, t, v, _ = synth.make_corpus(spec)
    ds = ref_dataset(ip, t, v, spec.dim)
    rng = np.random.default_rng(5)
    v2 = v * np.where(rng.random(v.size) < 0.3, -1.0, 1.0)
    ds2 = ref_dataset(ip, t, v2, spec.dim)
    # IVFD (variants.py:188-206): same similarities, its own label rule; signed
    # data makes the rule visible (objects whose best similarity is <= 0)
    dump("small_k32_ivfd", ds, 32, seed=23, max_iter=30, variant="IVFD")
    dump("signed_k16_ivfd", ds2, 16, seed=3, max_iter=20, variant="IVFD")
    # half the values negative and few means: many objects have no positive
    # similarity, so IVFD's "beat 0.0, else mean 1" rule decides their labels
    v3 = v * np.where(np.random.default_rng(9).random(v.size) < 0.5, -1.0, 1.0)
    dump("signed_k4_ivfd", ref_dataset(ip, t, v3, spec.dim), 4, seed=5, max_iter=15,
         variant="IVFD")
    if only_ivfd:
        return
    for k in (8, 32, 128):
        dump(f"small_k{k}", ds, k, seed=23, max_iter=30)
    # 2) signed values (the reference allows any finite nonzero value)
    dump("signed_k16", ds2, 16, seed=3, max_iter=20)
    # 3) duplicated rows -> duplicated means -> exact ties, empty (retained) clusters
    n0 = 300
    rows = rng.integers(0, n0 // 3, size=n0)
    parts_t, parts_v, cnt = [], [], []
    for r in rows:
        parts_t.append(t[ip[r]:ip[r + 1]])
        parts_v.append(v[ip[r]:ip[r + 1]])
        cnt.append(ip[r + 1] - ip[r])
    ip3 = np.zeros(n0 + 1, np.int64)
    np.cumsum(cnt, out=ip3[1:])
    ds3 = ref_dataset(ip3, np.concatenate(parts_t), np.concatenate(parts_v), spec.dim)
    dump("dups_k40", ds3, 40, seed=11, max_iter=20)
    # 4) config 0 at full size: outputs only (inputs regenerated by the generator)
    c0 = synth.CONFIGS[0]
    ip, t, v, _ = synth.make_corpus(c0["corpus"])
    ds0 = ref_dataset(ip, t, v, c0["corpus"].dim)
    dump("config0", ds0, c0["k"], seed=c0["seed"], max_iter=c0["iters"], store_inputs=False)


if __name__ == "__main__":
    main(only_ivfd="--ivfd" in sys.argv)
