"""The reference's OWN test suite, run through libopcfe from the reference's side.

integration/install.py installs the unmodified reference (baseline/_ref, built by
baseline/install_ref.sh from /root/reference/pkg) plus the libopcfe backend
(integration/flatpoly/_kernels/_opcfe.py: ctypes over include/opcfe.h, no torch) and
the maintainer's patch (integration/flatpoly_cuda.patch: the FLATPOLY_CUDA branch of
_kernels/__init__.py:9-30, mesh / FC functions routed to the backend).  With
FLATPOLY_CUDA=1 the reference's own tests -- tests/test_kernels.py (compiled backend vs
the NumPy fallback), test_smoothing.py, test_mesh.py, test_segmentation.py and
test_acceptance.py, test_accumulator.py (find_cells through the backend) and
test_stress.py (meshes of degenerate / noisy organized clouds) -- then exercise the GPU
kernels through the C ABI.

Deselected: acceptance #06 / #07 / #10 and one stress test run the polygon stage, which
needs the real Shapely (absent from this image; tests/golden/_stubs has an import stub
only) -- they fail identically on the stock reference here.
"""

import os
import subprocess
import sys

import pytest
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")
LIB = os.path.join(REPO, "paper_2007_12065_b200", "lib", "libopcfe.so")
STUBS = os.path.join(REPO, "tests", "golden", "_stubs")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device"),
              pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "flatpoly")),
                                 reason="baseline/_ref missing (run baseline/install_ref.sh)")]

FILES = ["tests/test_kernels.py", "tests/test_smoothing.py", "tests/test_mesh.py",
         "tests/test_segmentation.py", "tests/test_acceptance.py", "tests/test_accumulator.py",
         "tests/test_stress.py"]
DESELECT = ["tests/test_acceptance.py::test_06_room_benchmark",
            "tests/test_acceptance.py::test_07_thread_determinism",
            "tests/test_acceptance.py::test_10_buffer_geometry",
            "tests/test_stress.py::TestNoisyProjection::"
            "test_crossed_projection_passes_through_and_buffer_repairs"]


@pytest.fixture(scope="module")
def installed(tmp_path_factory):
    dest = str(tmp_path_factory.mktemp("flatpoly_cuda"))
    subprocess.run([sys.executable, os.path.join(REPO, "integration", "install.py"), dest],
                   check=True)
    return dest


def _env(dest, mode="1"):
    env = dict(os.environ, FLATPOLY_CUDA=mode, OPCFE_LIB=LIB,
               PYTHONPATH=os.pathsep.join([dest, STUBS]))
    env.pop("FLATPOLY_PURE", None)
    return env


def test_backend_is_libopcfe(installed):
    code = ("from flatpoly import _kernels, mesh\n"
            "import numpy as np\n"
            "assert _kernels.ACTIVE == 'cuda', _kernels.ACTIVE\n"
            "assert _kernels.laplacian_filter.__module__ == 'flatpoly._kernels._opcfe'\n"
            "mesh.mesh_from_opc(np.zeros((4, 4, 3)))\n"
            "maps = open('/proc/self/maps').read()\n"
            "assert 'libopcfe.so' in maps, 'libopcfe not mapped'\n"
            "print('ok')\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=installed, env=_env(installed),
                       capture_output=True, text=True)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_reference_suite_through_libopcfe(installed):
    args = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", *FILES]
    for d in DESELECT:
        args += ["--deselect", d]
    r = subprocess.run(args, cwd=installed, env=_env(installed), capture_output=True, text=True,
                       timeout=1200)
    tail = "\n".join(r.stdout.splitlines()[-25:])
    print(tail)
    assert r.returncode == 0, tail + r.stderr[-2000:]
    assert " passed" in tail and "failed" not in tail


CHAIN = r"""
import sys
import numpy as np
from flatpoly import _kernels, mesh, smoothing
from flatpoly.synthetic import room_scene
rng = np.random.default_rng(7)
opc = room_scene(n=96, noise=0.002, seed=3).opc
opc[rng.random(opc.shape[:2]) < 0.05] = np.nan
sm = smoothing.laplacian_filter_opc(opc, smoothing.LaplacianParams(0.8, 3, 4))
m = mesh.mesh_from_opc(sm)
n = smoothing.bilateral_filter_opc(sm, smoothing.BilateralParams(0.1, 0.2, 5, 3), m.trimap)
n2 = smoothing.bilateral_filter_opc(sm, smoothing.BilateralParams(0.1, 0.2, 3, 2))
he2 = mesh.extract_halfedges_opc(m.trimap, *sm.shape[:2])
bad = m.trimap.copy()
bad[np.flatnonzero(bad >= 0)[-1]] = 10 ** 9            # an out-of-range GID entry
try:
    smoothing.bilateral_filter_opc(sm, smoothing.BilateralParams(0.1, 0.2, 3, 1), bad)
    err = "none"
except Exception as e:
    err = type(e).__name__
np.savez(sys.argv[1], active=_kernels.ACTIVE, sm=sm, tri=m.triangles, he=m.halfedges,
         tm=m.trimap, mn=m.normals, n=n, n2=n2, he2=he2, err=err)
"""


def test_fused_binding_chain_equals_stock_native(installed, tmp_path):
    """The patch's fused mesh_from_opc / bilateral_filter_opc (one upload; gather on the
    device) against the same stock code on the reference's compiled CPU backend, incl. the
    IndexError of an out-of-range GID map (checked on the device: opcfe_trimap_stats)."""
    import numpy as np
    out = {}
    for mode in ("cuda", "native"):
        env = _env(installed)
        if mode == "native":
            env.pop("FLATPOLY_CUDA")
        path = str(tmp_path / f"{mode}.npz")
        r = subprocess.run([sys.executable, "-c", CHAIN, path], cwd=installed, env=env,
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-2000:]
        out[mode] = np.load(path)
        assert str(out[mode]["active"]) == mode
    g, r = out["cuda"], out["native"]
    assert str(g["err"]) == str(r["err"]) == "IndexError"
    for k in ("sm", "tri", "he", "tm", "mn", "he2"):
        assert g[k].shape == r[k].shape and np.array_equal(g[k], r[k], equal_nan=(k in ("sm", "mn"))), k
    for k in ("n", "n2"):
        bad = np.isnan(r[k]).any(1)
        assert np.array_equal(np.isnan(g[k]).any(1), bad), k
        assert np.abs(g[k][~bad] - r[k][~bad]).max() <= 1e-12, k
