"""Assign / update steps with the reference's signatures (variants.py), on B200.

* ``assign_ivf(ds, means, counters=None, backend=None, workspace=None)``
  <- variants.py:162-174: same checks (representation, dim, k, owner count),
  same result type (1-based ``Assignment``), counters gain V = postings
  touched in mults/adds/inner_entries exactly like _kernels.pyx:126-128.
* ``update_ivf(ds, asg, prev)`` <- variants.py:310-312 (update_means
  :254-307): bit-identical means, empty clusters retained.
* ``assign_ivfd(ds, means, ...)`` <- variants.py:188-206 (IVFD): the same
  exact similarities (both variants add the products in ascending term
  order), the IVFD label rule (an argmax must beat 0.0, else mean 1,
  _kernels.pyx:178-207); the object inverted file is not needed on the
  device (accepted and checked like the reference).
* ``update_sparse_standard`` <- variants.py:315-317 (IVFD's update).
* ``assign_step`` / ``update_step`` <- variants.py:219-234, 340-345 (IVF, IVFD).

The dataset is uploaded once and cached on the device by object identity
(the reference arrays are immutable), so repeated calls on the same Dataset
pay the host->device copy once.
"""

from __future__ import annotations

import weakref

import numpy as np
import torch

from .engine import DeviceDataset, DeviceMeans, LloydEngine
from .types import Assignment, CorruptionError, MeanSet, OpCounters

__all__ = ["assign_ivf", "assign_ivfd", "update_ivf", "update_sparse_standard", "assign_step",
           "update_step", "Workspace", "engine_for"]

_ENGINES: dict[int, tuple[LloydEngine, object]] = {}


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 path needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def engine_for(ds, k: int) -> LloydEngine:
    """Device engine for (ds, k), cached while ds is alive."""
    key = id(ds)
    hit = _ENGINES.get(key)
    if hit is not None and hit[0].k == k and hit[1]() is ds:
        return hit[0]
    eng = LloydEngine(DeviceDataset.from_dataset(ds, _device()), k)
    try:
        ref = weakref.ref(ds, lambda _r, key=key: _ENGINES.pop(key, None))
    except TypeError:  # not weak-referenceable: keep a strong reference
        ref = (lambda obj: (lambda: obj))(ds)
    _ENGINES[key] = (eng, ref)
    return eng


class Workspace:
    """variants.py:86-103 holds per-run host scratch; here the scratch lives in
    the device engine, so this is kept for signature compatibility."""


def _require(means, representation: str, variant: str) -> None:
    if means.representation != representation:
        raise ValueError(f"{variant} needs means in {representation!r} form, "
                         f"got {means.representation!r}")


def assign_ivf(ds, means, counters: OpCounters | None = None, backend: str | None = None,
               workspace: Workspace | None = None) -> Assignment:
    """Scan of the means' per-term postings (variants.py:162-174) on the GPU."""
    _require(means, "sparse_inverted", "IVF")
    return _assign(ds, means, counters, backend, rule=0)


def assign_ivfd(ds, means, counters: OpCounters | None = None, backend: str | None = None,
                workspace: Workspace | None = None, obj_inverted=None) -> Assignment:
    """IVFD assignment (variants.py:188-206) on the GPU: same similarities as
    IVF, the IVFD label rule (argmax only above 0.0, else mean 1)."""
    _require(means, "sparse_standard", "IVFD")
    if obj_inverted is not None and (obj_inverted.n_owners != ds.n
                                     or obj_inverted.dim != ds.dim):
        raise CorruptionError("object postings do not match the dataset")
    return _assign(ds, means, counters, backend, rule=1)


def _assign(ds, means, counters, backend, rule: int) -> Assignment:
    if ds.dim != means.dim:
        raise ValueError("dataset and means disagree on dim")
    if means.k < 1:
        raise ValueError("mean set is empty")
    if backend not in (None, "b200"):
        raise ValueError(f"unknown backend {backend!r}; choices: b200")
    if means.term_ids.size and (int(np.min(means.term_ids)) < 1
                                or int(np.max(means.term_ids)) > means.dim):
        raise CorruptionError("mean postings reference terms beyond dim")
    eng = engine_for(ds, means.k)
    dm = eng.upload_means(means)
    lab = eng.assign(dm, None, rule=rule)
    st = eng.read_stats()
    if counters is not None:
        counters.add_array([st.postings, st.postings, st.postings, 0, 0])
    labels = lab.cpu().numpy() + 1
    return Assignment(labels.astype(np.int32), eng.sizes.cpu().numpy().astype(np.int64))


def update_ivf(ds, asg, prev) -> MeanSet:
    """Update step emitting the means as per-term postings (variants.py:310-312)."""
    return _update(ds, asg, prev, "sparse_inverted")


def update_sparse_standard(ds, asg, prev) -> MeanSet:
    """Update step emitting per-mean sorted sparse vectors (variants.py:315-317)."""
    return _update(ds, asg, prev, "sparse_standard")


def _update(ds, asg, prev, representation: str) -> MeanSet:
    k = prev.k
    if asg.k != k or asg.n != ds.n:
        raise ValueError("assignment does not match dataset and means")
    eng = engine_for(ds, k)
    dm = DeviceMeans.from_meanset(prev, eng.device)
    lab = torch.from_numpy(np.ascontiguousarray(asg.labels, dtype=np.int32) - 1).to(eng.device)
    eng.sizes.copy_(torch.from_numpy(np.array(asg.sizes, dtype=np.int64)))
    new = eng.update(lab, dm)
    return new.to_meanset(representation)


def assign_step(variant, ds, means, counters=None, backend=None, workspace=None,
                obj_inverted=None) -> Assignment:
    if variant == "IVFD":
        return assign_ivfd(ds, means, counters, backend, workspace, obj_inverted)
    if variant != "IVF":
        raise ValueError(f"unknown variant {variant!r} on the B200 path")
    return assign_ivf(ds, means, counters, backend, workspace)


def update_step(variant, ds, asg, prev) -> MeanSet:
    if variant == "IVFD":
        return update_sparse_standard(ds, asg, prev)
    if variant != "IVF":
        raise ValueError(f"unknown variant {variant!r} on the B200 path")
    return update_ivf(ds, asg, prev)
