"""pytest plugin: run the reference's own backend-parametrised test suite
with this repository's B200 kernels registered as backend ``"b200"``.

The reference selects its hot loop through a registry of kernel modules
(/root/reference/pkg/src/sparse_kmeans/kernels.py:23-52) and parametrises
its tests over ``available_backends()`` at collection time
(/root/reference/pkg/tests/conftest.py:52-54).  Loading this plugin with
``pytest -p b200_plugin`` — before the reference's conftest is imported —
adds the entry, so every test that takes the ``backend`` fixture also runs
``run(..., backend="b200")`` / ``assign_ivf(..., backend="b200")`` on the GPU
(no edit to the reference).

The registered module is ``paper_2002_09094_b200.backend`` (IVF and IVFD on
the B200 path, through the C ABI ``ivfkm_assign_ivf_host`` /
``ivfkm_assign_ivfd_host``) plus the comparison variants MFN/IFN/IFB/TWM,
which are outside the B200 path and are delegated to the
reference's compiled module (numpy module when it is not built), so those
tests exercise the registration without claiming the GPU ran them.

Without a CUDA device the ``b200`` cases are skipped (collection still shows
them), so the plugin can be checked on a CPU-only host.

Usage: tools/refsuite/run_reference_suite.sh
"""

from __future__ import annotations

import sys
import types
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[2]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

import sparse_kmeans.kernels as K  # noqa: E402  (the reference package under test)

from paper_2002_09094_b200 import backend as _b200  # noqa: E402


def _module():
    other = K._MODULES.get("compiled") or K._MODULES["python"]
    m = types.ModuleType("b200_kernels")
    m.BACKEND_NAME = "b200"
    m.assign_ivf = _b200.assign_ivf
    m.assign_ivfd = _b200.assign_ivfd
    for name in ("assign_mfn", "assign_ifn", "assign_ifb", "assign_twm"):
        setattr(m, name, getattr(other, name))
    return m


K._MODULES["b200"] = _module()


def _have_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _have_gpu():
        return
    skip = pytest.mark.skip(reason="backend b200 needs a CUDA device")
    for it in items:
        cs = getattr(it, "callspec", None)
        if cs is not None and cs.params.get("backend") == "b200":
            it.add_marker(skip)
