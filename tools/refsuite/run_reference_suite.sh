#!/usr/bin/env bash
# Run the reference's own test suite with the B200 kernels registered as
# backend "b200" (tools/refsuite/b200_plugin.py).  Needs the reference tree
# (REF_ROOT, default /root/reference; read only: it is copied to a scratch
# directory and its Cython kernel built there, as pkg/setup.py does) and, for
# the b200 cases to run rather than skip, a CUDA device.
#   tools/refsuite/run_reference_suite.sh [extra pytest args, e.g. -k b200]
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REPO="$(cd "$HERE/../.." && pwd)"
REF="${REF_ROOT:-/root/reference}/pkg"
[ -d "$REF" ] || { echo "no reference tree at $REF" >&2; exit 2; }
WORK="$(mktemp -d /tmp/refsuite.XXXXXX)"
cp -r "$REF" "$WORK/pkg"
(cd "$WORK/pkg" && python setup.py build_ext --inplace >/dev/null 2>&1) || \
  echo "reference extension not built; its numpy backend stands in" >&2
cd "$WORK/pkg"
PYTHONPATH="$WORK/pkg/src:$HERE:$REPO" python -m pytest -p b200_plugin tests -q "$@"
