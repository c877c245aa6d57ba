"""The reference's own backend-parametrised suite with the B200 module
registered as backend "b200" (tools/refsuite): where the reference tree is
present (this build container) the plugin must load, register, and add the
b200 cases (run on a GPU host, skipped on a CPU-only one) without breaking
any of the reference's own cases."""

import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg")


@pytest.mark.skipif(not REF.is_dir(), reason="reference tree not present")
def test_reference_suite_runs_with_b200_backend_registered():
    res = subprocess.run(["bash", str(ROOT / "tools" / "refsuite" / "run_reference_suite.sh"),
                          "-rs"], capture_output=True, text=True, timeout=900)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-3000:]
    m = re.search(r"(\d+) passed", out)
    assert m and int(m.group(1)) >= 150, out[-2000:]
    b200 = re.findall(r"\[b200", out) + re.findall(r"b200 needs a CUDA device", out)
    assert b200, "no b200-parametrised case was collected"
