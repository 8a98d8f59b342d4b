#!/bin/bash
# Copy the reference's own test files (unchanged) next to the baseline/_ref
# install, so tests/test_reference_suite.py can run them on the GPU box, where
# /root/reference does not exist. baseline/_ref_tests is git-ignored (like
# baseline/_ref): it is never committed, only shipped with the gpurun snapshot.
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=${1:-/root/reference/pkg/tests}
mkdir -p "$ROOT/baseline/_ref_tests"
for f in test_pack.py test_acceptance.py test_tuner.py test_data.py; do
  cp "$SRC/$f" "$ROOT/baseline/_ref_tests/$f"
done
ls -l "$ROOT/baseline/_ref_tests"
