#!/usr/bin/env bash
# Install the UNMODIFIED reference (rfsplat, pure Python) into baseline/_ref
# (git-ignored; it travels to the GPU box with the gpurun snapshot).  Also
# places the reference's own test suite beside it (baseline/_ref/rfsplat_tests)
# so tests/test_gpu_reference_suite.py can run it against the drop-in on a box
# where /root/reference does not exist.  Nothing is copied into tracked files.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
DEST="$ROOT/baseline/_ref"
if [ ! -d "$SRC" ]; then
  echo "reference not present at $SRC; nothing to install" >&2
  exit 0
fi
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"   # the reference tree is read-only; build from a copy
rm -rf "$DEST"
python -m pip install --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$DEST" "$TMP/pkg" >/dev/null
cp -r "$SRC/tests" "$DEST/rfsplat_tests"
echo "installed rfsplat into $DEST"
