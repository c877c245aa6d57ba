#!/usr/bin/env bash
# ORACLE — test infrastructure only.  Compiles the reference's own hot-loop
# module (/root/reference/pkg/src/sparse_kmeans/_kernels.pyx, built by the
# reference with Cython + "-O3", pkg/setup.py:9-13) into oracle/_ref/ so the
# CPU baseline and the parity tests can run the *reference* kernel, not only
# the restatement.  Outputs go to oracle/_ref/ only (git-ignored; it travels
# to the GPU box with the snapshot).  No reference source is copied into the
# repository; the generated C lives in oracle/_ref/ next to the .so.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${REF_ROOT:-/root/reference}/pkg/src/sparse_kmeans/_kernels.pyx"
OUT="$HERE/_ref"
if [ ! -f "$SRC" ]; then
  echo "reference source $SRC not present; skipping oracle/_ref" >&2
  exit 0
fi
mkdir -p "$OUT"
PY="${PYTHON:-python3}"
"$PY" -m cython -3 -o "$OUT/_kernels.c" "$SRC"
INC="$("$PY" -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
SUF="$("$PY" -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
gcc -O3 -fPIC -shared -I"$INC" -o "$OUT/_kernels$SUF" "$OUT/_kernels.c"
echo "$OUT/_kernels$SUF"
