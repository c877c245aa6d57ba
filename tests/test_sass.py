"""SASS guards for the screen's hot loop (cuobjdump on the built library, no
GPU needed).  ptxas' scheduling of the dense-prefix loop is fragile: a change
elsewhere in the kernel once made it sink the loads next to their uses — two
loads in flight instead of four, 17% slower at config 1.  These checks pin
the property the kernel's speed rests on, and that the hardware paths are
the intended ones (FFMA2, 128-bit constant-cache loads)."""

import re
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
OBJ = ROOT / "paper_2002_09094_b200" / "_lib" / "obj" / "assign.cu.o"


def _sass(fn_pattern):
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(tool).exists() or not OBJ.exists():
        pytest.skip("cuobjdump or the built object missing")
    names = subprocess.run([tool, "-sass", str(OBJ)], capture_output=True, text=True).stdout
    fns = [m for m in re.findall(r"Function : (\S+)", names) if re.search(fn_pattern, m)]
    assert fns, fn_pattern
    out = subprocess.run([tool, "-sass", "-fun", fns[0], str(OBJ)], capture_output=True,
                         text=True).stdout
    return [m.group(1) for m in re.finditer(r"/\*[0-9a-f]{4}\*/\s+(.*?);", out)]


# (instantiation, loads in flight before the first use): the 56-register
# small-CTA screen runs every production plan; the 64-register one only the
# forced one-pass plans and the DSMEM cluster split
@pytest.mark.parametrize("inst,need", [("ILi8ELb1ELi56E", 4), ("ILi8ELb1ELi64E", 3)])
def test_dense_loop_keeps_loads_in_flight(inst, need):
    ops = _sass(r"screen_kernel" + inst)
    first_use = next(i for i, o in enumerate(ops) if "HADD2.F32" in o)
    before = [o for o in ops[max(0, first_use - 40):first_use] if "LDG.E.128" in o]
    assert len(before) >= need, f"{len(before)} dense loads issued before the first use"
    assert any("FFMA2" in o for o in ops) or inst.endswith("64E")
