import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")
    # the C-ABI library and the C oracle are built in-tree; build them if stale
    from paper_2002_09094_b200 import build as B

    if B._stale():
        B.build_library()
    from oracle import oracle as O

    O.build()


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def load_golden(name):
    return dict(np.load(GOLDEN / f"{name}.npz", allow_pickle=False))


R = 2 ** -0.5


@pytest.fixture
def tiny():
    """The reference's worked example (conftest.py:10-16): x1={1,2}, x2={2,3}, x3={3,4}."""
    from paper_2002_09094_b200 import Dataset

    indptr = np.array([0, 2, 4, 6], np.int64)
    terms = np.array([1, 2, 2, 3, 3, 4], np.int32)
    vals = np.full(6, R)
    return Dataset(4, indptr, terms, vals, normalized=True)


@pytest.fixture
def tiny_means():
    """conftest.py:19-25: mu1 = normalized(x1 + x2) = (s, 2s, s, 0), mu2 = x3."""
    from paper_2002_09094_b200 import MeanSet

    s = 6 ** -0.5
    return MeanSet.from_csr(np.array([0, 3, 5], np.int64), np.array([1, 2, 3, 3, 4], np.int32),
                            np.array([s, 2 * s, s, R, R]), 4, "sparse_inverted")


def golden_dataset(g):
    from paper_2002_09094_b200 import Dataset

    return Dataset(int(g["dim"]), g["indptr"], g["term_ids"], g["values"], normalized=True)
