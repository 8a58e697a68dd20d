#!/bin/bash
# Installs the unmodified reference package (svdlut, /root/reference/pkg) into
# the git-ignored baseline/_ref/ (it travels to the GPU box with gpurun), plus
# a copy of the reference's own test suite in baseline/_ref/svdlut_tests/ for
# tests/test_gpu_reference_suite.py (the drop-in run on the B200).  The build
# runs from a copy under /tmp: /root/reference is read-only.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "reference not present at $SRC" >&2; exit 1; }
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" "$TMP/pkg" >/dev/null
cp -r "$SRC/tests" "$ROOT/baseline/_ref/svdlut_tests"
rm -rf "$TMP"
echo "installed svdlut into $ROOT/baseline/_ref"
