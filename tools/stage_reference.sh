#!/bin/bash
# Stages the unmodified reference for the compatibility shim (compat/powersort)
# and its test-suite run (tests/test_reference_suite.py):
#   baseline/_ref/powersort   -- pip install --target of /root/reference (offline)
#   baseline/_ref/ref_tests   -- a copy of /root/reference/pkg/tests
# baseline/_ref is git-ignored (never committed) but travels to the GPU box.
set -e
REPO=$(cd "$(dirname "$0")/.." && pwd)
REF=${REF:-/root/reference}
OUT=$REPO/baseline/_ref
mkdir -p "$OUT"
if [ ! -d "$OUT/powersort" ]; then
  TMP=$(mktemp -d)
  cp -r "$REF/pkg" "$TMP/pkg"
  python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
      --target "$OUT" "$TMP/pkg" > "$OUT/pip.log" 2>&1 || { echo "pip install failed, see $OUT/pip.log"; exit 1; }
  rm -rf "$TMP"
fi
rm -rf "$OUT/ref_tests"
cp -r "$REF/pkg/tests" "$OUT/ref_tests"
echo "staged: $(ls "$OUT")"
