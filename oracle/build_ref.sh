#!/usr/bin/env bash
# Build the REFERENCE's own compiled kernels (flatpoly/_kernels/_native.pyx) from
# the sources where they lie under /root/reference, into oracle/_ref/ (git-ignored,
# NOT gpurun-ignored, so the .so travels to the GPU box as the CPU baseline).
#
# Test/bench infrastructure only: the product path never loads this module.
# Recipe mirrors the reference's own setup.py:17-29 flags (-O3 -ffp-contract=off);
# we do not run the reference's build system (setuptools), just cython + gcc.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${REF_ROOT:-/root/reference}/pkg/src/flatpoly/_kernels/_native.pyx"
OUT="$HERE/_ref"
if [ ! -f "$SRC" ]; then
  echo "reference source not found ($SRC); keeping prebuilt oracle/_ref" >&2
  exit 0
fi
mkdir -p "$OUT"
PY="${PYTHON:-python}"
PYINC="$($PY -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
NPINC="$($PY -c 'import numpy; print(numpy.get_include())')"
# cython writes only into oracle/_ref (the .pyx is read in place, read-only)
$PY -m cython -3 --module-name _native -o "$OUT/_native.c" "$SRC"
gcc -shared -fPIC -O3 -ffp-contract=off -I"$PYINC" -I"$NPINC" \
    -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION \
    "$OUT/_native.c" -o "$OUT/_native.so" -lm
echo "built $OUT/_native.so"
