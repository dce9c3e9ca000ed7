#!/bin/sh
# Installs the UNMODIFIED reference package (pure Python + numpy) into baseline/_ref
# (git-ignored, shipped to the GPU box by gpurun).  The source tree is read-only,
# so pip builds from a copy; numpy is already in the image, so dependency
# resolution is skipped (--no-deps).  Used by bench.py --impl reference and by
# tests/test_gpu_ref_protocol.py.
set -e
here=$(cd "$(dirname "$0")" && pwd)
src=${1:-/root/reference/pkg}
tmp=$(mktemp -d)
cp -r "$src" "$tmp/pkg"
rm -rf "$here/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$here/_ref" "$tmp/pkg"
rm -rf "$tmp"
