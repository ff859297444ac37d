#!/usr/bin/env bash
# Install the unmodified reference package (tmfgclust) into baseline/_ref with the offline wheelhouse,
# and put its unmodified test suite beside it (baseline/_ref/tests).  baseline/_ref is git-ignored and
# travels to the GPU box with the gpurun snapshot; tests/test_gpu_dropin.py and bench.py read it there.
# The build writes into its source tree, so it installs from a copy under /tmp (/root/reference is read-only).
set -euo pipefail
REPO="$(cd "$(dirname "$0")/.." && pwd)"
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d /tmp/tg_refsrc.XXXX)
cp -r "$SRC"/. "$TMP"/
rm -rf "$REPO/baseline/_ref"
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
    --target "$REPO/baseline/_ref" "$TMP"
mkdir -p "$REPO/baseline/_ref/tests"
cp "$SRC"/tests/*.py "$REPO/baseline/_ref/tests/"
rm -rf "$TMP"
echo "installed: $(ls "$REPO/baseline/_ref")"
