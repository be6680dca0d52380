#!/usr/bin/env bash
# Installs the UNMODIFIED reference package (pkg/src/batchrand) into baseline/_ref so that
# tests/test_refbind.py and bench.py's context fields can import it on the GPU box, where
# /root/reference does not exist.  baseline/_ref is git-ignored but travels with gpurun.
# The build writes into its source tree, so it runs from a copy under /tmp (the reference is
# read-only); the package has no runtime dependencies (pyproject.toml:10).
set -euo pipefail
REPO="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference}/pkg"
[ -f "$SRC/pyproject.toml" ] || { echo "no reference package at $SRC" >&2; exit 1; }
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$REPO/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$REPO/baseline/_ref" "$TMP/pkg"
python -c "import sys; sys.path.insert(0, '$REPO/baseline/_ref'); import batchrand; print('vendored', batchrand.__file__)"
