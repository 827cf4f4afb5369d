#!/bin/sh
# Stages the unmodified reference (pure Python, /root/reference/pkg) for the
# GPU box, where /root/reference does not exist.  Everything goes under
# baseline/_ref/, which is git-ignored (never committed) but travels with
# gpurun snapshots:
#   baseline/_ref/genopt/            the installed package (bench.py --impl reference)
#   baseline/_ref/reference_pkg/tests/  its own test suite + fixtures, run against this
#                                    package by tests/test_gpu_reference_api.py
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
rm -rf /tmp/genopt_build "$ROOT/baseline/_ref"
cp -r "$SRC" /tmp/genopt_build
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" /tmp/genopt_build
mkdir -p "$ROOT/baseline/_ref/reference_pkg"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/reference_pkg/tests"
echo "staged reference into $ROOT/baseline/_ref"
