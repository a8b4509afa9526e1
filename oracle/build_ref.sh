#!/usr/bin/env bash
# Install the REFERENCE package (pure Python "tokenflow") into oracle/_ref so
# bench.py's reference arm and the CPU baseline can run the reference's own
# engines on the GPU box (/root/reference does not exist there).  Built from a
# /tmp copy because the reference tree is read-only; oracle/_ref is
# git-ignored (not copied into history) but travels with the gpurun snapshot.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${PRUNE_REFERENCE:-/root/reference/pkg}"
[ -d "$SRC" ] || { echo "reference not present at $SRC; skipping"; exit 0; }
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$HERE/_ref" "$TMP/pkg"
rm -rf "$TMP"
echo "reference installed into $HERE/_ref"
