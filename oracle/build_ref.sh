#!/bin/sh
# Installs the UNMODIFIED reference package `phaseswe` (pure Python on
# numpy/scipy, /root/reference/pkg) into oracle/_ref with pip's own build of
# the package -- the Python analogue of compiling a C reference into
# oracle/_ref.  oracle/_ref is git-ignored (no reference sources enter the
# history) but not gpurun-ignored, so the reference travels to the GPU box,
# where bench.py's CPU legs time it (cpu_baseline.kind = "reference") and
# check the GPU result against it.  Test infrastructure only.
set -e
SRC=${1:-/root/reference/pkg}
HERE=$(cd "$(dirname "$0")" && pwd)
[ -d "$SRC" ] || { echo "reference not found at $SRC; oracle/_ref not built"; exit 0; }
TMP=$(mktemp -d)
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"            # the reference tree is read-only; setuptools writes build/ into it
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --target "$HERE/_ref" "$TMP/pkg"
python -c "import sys; sys.path.insert(0, '$HERE/_ref'); import phaseswe; print('oracle/_ref: phaseswe', phaseswe.__file__)"
