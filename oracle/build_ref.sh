#!/usr/bin/env bash
# Build the REFERENCE's own kernel module from its source where it lies
# (/root/reference/pkg/src/filterkit/_ckernels.pyx) into oracle/_ref/
# (git-ignored; it travels to the GPU box as a built .so).  Same recipe as
# the reference's pkg/setup.py:10-16: Cython, then the C compiler at -O3
# with numpy's headers.  The generated C file is deleted after compiling --
# only the binary is kept.  Used as the CPU baseline ("kind": "reference")
# and as a second checker for the oracle restatement.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC=/root/reference/pkg/src/filterkit/_ckernels.pyx
OUT="$HERE/_ref"
[ -f "$SRC" ] || { echo "reference source not present; skipping oracle/_ref"; exit 0; }
PY=${PYTHON:-python}
SUFFIX=$($PY -c "import sysconfig; print(sysconfig.get_config_var('EXT_SUFFIX'))")
TARGET="$OUT/_ckernels$SUFFIX"
if [ -f "$TARGET" ] && [ "$TARGET" -nt "$SRC" ]; then echo "oracle/_ref up to date"; exit 0; fi
mkdir -p "$OUT"
TMP=$(mktemp -d)
cp "$SRC" "$TMP/_ckernels.pyx"
$PY -m cython -3 "$TMP/_ckernels.pyx" -o "$TMP/_ckernels.c"
NPINC=$($PY -c "import numpy; print(numpy.get_include())")
PYINC=$($PY -c "import sysconfig; print(sysconfig.get_paths()['include'])")
gcc -O3 -shared -fPIC -I"$PYINC" -I"$NPINC" "$TMP/_ckernels.c" -o "$TARGET"
rm -rf "$TMP"
echo "built $TARGET"
