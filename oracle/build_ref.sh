#!/usr/bin/env bash
# Build the reference's only native component, _native_ops.pyx, out of tree
# (SURVEY.md 8(c) "path 2") into oracle/_ref/.  Test/baseline infrastructure:
# the output is used only as a CPU checker and as bench.py's reference arm.
# Compiled from the source where it lies under /root/reference (never copied
# into the repo); intermediate C is deleted.  -march=native from the
# reference's setup.py:8 is replaced by x86-64-v3 so the .so runs on the GPU
# box's host too (checked at load time, see oracle/ref_ops.py).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC=/root/reference/pkg/src/depthfill/_native_ops.pyx
OUT="$HERE/_ref"
[ -f "$SRC" ] || { echo "reference not present; skipping oracle/_ref build"; exit 0; }
mkdir -p "$OUT"
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
PY=${PYTHON:-python}
"$PY" -m cython -3 "$SRC" -o "$TMP/_native_ops.c"
EXT=$("$PY" -c 'import sysconfig;print(sysconfig.get_config_var("EXT_SUFFIX"))')
INC=$("$PY" -c 'import sysconfig;print(sysconfig.get_paths()["include"])')
NPINC=$("$PY" -c 'import numpy;print(numpy.get_include())')
gcc -O3 -march=x86-64-v3 -fno-math-errno -shared -fPIC -I"$INC" -I"$NPINC" \
    "$TMP/_native_ops.c" -o "$OUT/_native_ops$EXT"
echo "built $OUT/_native_ops$EXT"
