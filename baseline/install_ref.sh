#!/usr/bin/env bash
# Install the UNMODIFIED reference (flatpoly, /root/reference/pkg) into baseline/_ref
# (git-ignored, NOT gpurun-ignored: it travels to the GPU box) -- the base contract's
# offline install, from a /tmp copy because setuptools writes build files into the
# source tree (/root/reference is read-only).  --no-deps: numpy / scipy are in the
# image, shapely is absent (the hot path never calls it; tests/golden/_stubs has an
# import stub).  The reference's own tests are copied alongside (baseline/_ref/pkg_tests)
# so the GPU box can run them through libopcfe (tests/test_gpu_reference_suite.py).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${REF_ROOT:-/root/reference}/pkg"
if [ ! -d "$SRC" ]; then
  echo "reference not found ($SRC); keeping the existing baseline/_ref" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/flatpoly_src.XXXXXX)"
cp -r "$SRC/." "$TMP/"
rm -rf "$HERE/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$HERE/_ref" "$TMP" > "$HERE/install_ref.log" 2>&1
cp -r "$SRC/tests" "$HERE/_ref/pkg_tests"
rm -rf "$TMP"
python - <<PY
import sys; sys.path[:0] = ["$HERE/_ref", "$HERE/../tests/golden/_stubs"]
from flatpoly import _kernels
assert _kernels.ACTIVE == "native", _kernels.ACTIVE
print("baseline/_ref: flatpoly installed, kernel backend", _kernels.ACTIVE)
PY
