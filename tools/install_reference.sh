#!/bin/bash
# Install the UNMODIFIED reference (gmfkit, with its compiled Cython kernel)
# into baseline/_ref for bench.py --impl reference.  /root/reference is
# read-only, so the build runs from a copy under /tmp.  baseline/_ref is
# git-ignored but travels to the GPU box with the repo snapshot.
set -e
REPO="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no $SRC: keeping any existing baseline/_ref"; exit 0; }
TMP="$(mktemp -d /tmp/gmfkit_src.XXXXXX)"
cp -r "$SRC"/. "$TMP"/
rm -rf "$REPO/baseline/_ref"
mkdir -p "$REPO/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$REPO/baseline/_ref" "$TMP" 
rm -rf "$TMP"
PYTHONPATH="$REPO/baseline/_ref" python -c "import gmfkit.kernels as k; print('gmfkit kernels.IMPL =', k.IMPL)"
