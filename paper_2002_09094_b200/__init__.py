"""B200-native IVF spherical k-means (arXiv 2002.09094), drop-in for the
reference package's IVF Lloyd path.

Public API mirrors ``sparse_kmeans`` (reference clustering.py / variants.py /
data.py / means.py): ``run``, ``init_means``, ``assign_ivf``, ``update_ivf``,
``objective_cosine``, ``Dataset``, ``MeanSet``, ``Assignment``,
``OpCounters``, ``RunResult``.  The hot path runs in libivfkm.so (hand-written
sm_100a CUDA behind the C ABI in include/ivfkm.h); there is no CPU fallback.
"""

from .types import (  # noqa: F401
    COUNTER_FIELDS, Assignment, CorruptionError, Dataset, MeanSet, OpCounters, fnv1a64,
)

__all__ = [
    "Dataset", "MeanSet", "Assignment", "OpCounters", "CorruptionError", "fnv1a64",
    "run", "fit", "init_means", "objective_cosine", "assign_ivf", "update_ivf",
    "assign_step", "update_step", "RunResult", "IterationRecord", "SplitMix64",
    "sample_without_replacement",
]


def __getattr__(name):  # lazy: importing the types must not require torch / the .so
    if name in ("run", "fit", "init_means", "objective_cosine", "RunResult", "IterationRecord",
                "SplitMix64", "sample_without_replacement"):
        from . import clustering
        return getattr(clustering, name)
    if name in ("assign_ivf", "update_ivf", "assign_step", "update_step", "Workspace"):
        from . import variants
        return getattr(variants, name)
    raise AttributeError(name)
