#!/usr/bin/env python
"""Install flatpoly with the libopcfe backend into DEST -- what a maintainer does once.

    python integration/install.py DEST [--ref baseline/_ref]

1. copies the installed reference package (baseline/_ref/flatpoly, built by
   baseline/install_ref.sh from /root/reference/pkg) and its tests (pkg_tests) into DEST;
2. adds integration/flatpoly/_kernels/_opcfe.py next to _native.pyx;
3. applies integration/flatpoly_cuda.patch: the FLATPOLY_CUDA branch of the kernel switch
   (_kernels/__init__.py:9-30), the mesh / FC functions routed to the backend
   (mesh.py:58,99,162; smoothing.py:61), and the two places that name the compiled
   backend explicitly (bench_kernels.py, tests/test_kernels.py).

Then:  FLATPOLY_CUDA=1 OPCFE_LIB=.../libopcfe.so PYTHONPATH=DEST python -m pytest DEST/tests
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)


def install(dest: str, ref: str) -> None:
    src_pkg = os.path.join(ref, "flatpoly")
    src_tests = os.path.join(ref, "pkg_tests")
    if not os.path.isdir(src_pkg):
        raise SystemExit(f"{src_pkg} missing: run baseline/install_ref.sh first")
    os.makedirs(dest, exist_ok=True)
    shutil.copytree(src_pkg, os.path.join(dest, "flatpoly"), dirs_exist_ok=True,
                    ignore=shutil.ignore_patterns("__pycache__"))
    if os.path.isdir(src_tests):
        shutil.copytree(src_tests, os.path.join(dest, "tests"), dirs_exist_ok=True,
                        ignore=shutil.ignore_patterns("__pycache__"))
    shutil.copy(os.path.join(HERE, "flatpoly", "_kernels", "_opcfe.py"),
                os.path.join(dest, "flatpoly", "_kernels", "_opcfe.py"))
    patch = os.path.join(HERE, "flatpoly_cuda.patch")
    subprocess.run(["git", "apply", "-p1", "--whitespace=nowarn", patch], cwd=dest, check=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("dest")
    ap.add_argument("--ref", default=os.path.join(REPO, "baseline", "_ref"))
    a = ap.parse_args()
    install(a.dest, a.ref)
    print(f"flatpoly + libopcfe backend installed in {a.dest}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
