#!/bin/bash
# Install the UNMODIFIED reference package into baseline/_ref (git-ignored, not
# gpurun-ignored: it travels to the GPU box) from a /tmp copy of
# /root/reference/pkg, plus its own test files under baseline/_ref/salf_tests
# (run against the B200 backend by tests/test_dropin_reference.py).  Dependency
# resolution is skipped (--no-deps): numpy / scipy are already in the image.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no reference at $SRC"; exit 0; }
rm -rf /tmp/salf_refsrc "$ROOT/baseline/_ref"
cp -r "$SRC" /tmp/salf_refsrc
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" /tmp/salf_refsrc
mkdir -p "$ROOT/baseline/_ref/salf_tests"
cp "$SRC"/tests/*.py "$ROOT/baseline/_ref/salf_tests/"
echo "installed reference into $ROOT/baseline/_ref"
