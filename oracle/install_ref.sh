#!/usr/bin/env bash
# Install the UNMODIFIED reference package (/root/reference/pkg: its Python
# facades + the Cython _ckernels built by its own setup.py) into
# baseline/_ref with pip, from a copy under /tmp (the reference tree is
# read-only), and copy its test suite (pkg/tests, unmodified) next to it as
# baseline/_ref/ref_tests.  baseline/ is git-ignored and travels to the GPU
# box with the snapshot, where /root/reference does not exist:
#   * bench.py --impl reference and the cpu_baseline legs drive this package
#     through its public API;
#   * tests/test_reference_suite_gpu.py runs ref_tests against the B200
#     build (the reference facades on our kernel contract, and our facades
#     under the name `filterkit`).
# Nothing here is product code and nothing is committed.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(dirname "$HERE")"
SRC=/root/reference/pkg
OUT="$ROOT/baseline/_ref"
[ -d "$SRC" ] || { echo "reference tree not present; skipping baseline/_ref"; exit 0; }
PY=${PYTHON:-python}
if [ -d "$OUT/filterkit" ] && [ -d "$OUT/ref_tests" ] && \
   [ -z "$(find "$SRC" -newer "$OUT/filterkit/__init__.py" -type f -print -quit)" ]; then
  echo "baseline/_ref up to date"; exit 0
fi
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$OUT"
mkdir -p "$OUT"
(cd "$TMP" && $PY -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
   --target "$OUT" "$TMP/pkg" > "$TMP/pip.log" 2>&1) || { cat "$TMP/pip.log"; exit 1; }
rm -f "$OUT/filterkit/_ckernels.c"
cp -r "$SRC/tests" "$OUT/ref_tests"
rm -rf "$TMP"
$PY -c "import sys; sys.path.insert(0, '$OUT'); import filterkit; assert filterkit.available_backends() == ['c', 'py']"
echo "installed the reference package into $OUT (backends c, py) + ref_tests"
