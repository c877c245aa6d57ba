"""Compile the sm_100a C-ABI library libivfkm.so in-tree with nvcc.

The library is plain CUDA C++ behind ``include/ivfkm.h`` (no torch types);
the package loads it with ctypes (``_lib.py``).
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libivfkm.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-fopenmp,-O3", "-Xptxas", "-v",
]


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))


def _stale() -> bool:
    if not LIB.exists():
        return True
    mt = LIB.stat().st_mtime
    deps = sources() + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "ivfkm.h"]
    return any(p.stat().st_mtime > mt for p in deps)


def _compile(src: Path, nvcc: str):
    """One translation unit -> _lib/obj/<name>.o (rebuilt when older than its
    source, any header or this file)."""
    obj = LIBDIR / "obj" / (src.name + ".o")
    hdrs = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [ROOT / "include" / "ivfkm.h",
                                                                  Path(__file__)]
    if obj.exists() and all(p.stat().st_mtime <= obj.stat().st_mtime for p in [src, *hdrs]):
        return obj, None
    cmd = [nvcc, *ARCH, *NVCC_FLAGS, "-I", str(ROOT / "include"), "-c", "-o", str(obj), str(src)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    return obj, (cmd, res)


def build_library(force: bool = False, verbose: bool = False) -> Path:
    """Compile each source in parallel (nvcc -c), then link the shared library."""
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    LIBDIR.mkdir(exist_ok=True)
    (LIBDIR / "obj").mkdir(exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    if force:
        for o in (LIBDIR / "obj").glob("*.o"):
            o.unlink()
    srcs = sources()
    with ThreadPoolExecutor(max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        results = list(ex.map(lambda s: _compile(s, nvcc), srcs))
    log = LIBDIR / "build.log"
    text = []
    for obj, r in results:
        if r is None:
            continue
        cmd, res = r
        text.append(" ".join(cmd) + "\n" + res.stdout + res.stderr)
        if res.returncode != 0:
            log.write_text("\n".join(text))
            sys.stderr.write(res.stderr[-6000:])
            raise RuntimeError(f"nvcc failed ({res.returncode}) on {cmd[-1]}; see {log}")
    cmd = [nvcc, *ARCH, "-shared", "-Xcompiler", "-fopenmp", "-o", str(LIB),
           *[str(o) for o, _ in results], "-lgomp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    text.append(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    log.write_text("\n".join(text))
    if res.returncode != 0:
        sys.stderr.write(res.stderr[-6000:])
        raise RuntimeError(f"nvcc link failed ({res.returncode}); see {log}")
    if verbose:
        sys.stderr.write("\n".join(text))
    return LIB


CORPUS_LIB = ROOT / "tools" / "_build" / "libcorpus.so"


def build_corpus_library(force: bool = False) -> Path:
    """The seeded corpus generator alone (csrc/synth.cpp, host C++/OpenMP, no
    CUDA): the reference arm of bench.py generates its inputs with it, so
    the reference's process never maps libivfkm.so."""
    src = CSRC / "synth.cpp"
    if not force and CORPUS_LIB.exists() and CORPUS_LIB.stat().st_mtime >= src.stat().st_mtime:
        return CORPUS_LIB
    CORPUS_LIB.parent.mkdir(parents=True, exist_ok=True)
    cxx = os.environ.get("CXX", "g++")
    obj = CORPUS_LIB.with_suffix(".o")
    res = subprocess.run([cxx, "-O3", "-std=c++17", "-fPIC", "-fopenmp", "-I",
                          str(ROOT / "include"), "-c", "-o", str(obj), str(src)],
                         capture_output=True, text=True)
    if res.returncode == 0:
        res = subprocess.run([cxx, "-shared", "-o", str(CORPUS_LIB), str(obj), "-l:libgomp.so.1"],
                             capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stderr[-4000:])
        raise RuntimeError("g++ failed on csrc/synth.cpp")
    return CORPUS_LIB


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose=True))
