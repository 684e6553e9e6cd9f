"""The drop-in API against the REAL reference, in process, on random inputs.

The stock reference (baseline/_ref: the unmodified flatpoly package with its compiled
Cython kernels, installed by baseline/install_ref.sh / __graft_entry__.build()) runs
pipeline.py:125-134's organized chain on random organized clouds beside this package's
drop-in functions at strict precision (the default for float64 input):

    sm = laplacian_filter_opc(opc, LaplacianParams)          smoothing.py:53
    mesh = mesh_from_opc(sm)                                  mesh.py:167
    mesh.normals = bilateral_filter_opc(sm, BilateralParams, mesh.trimap)
    labels = group_assignment(mesh, dominant, l_max, ang_min) segmentation.py:52

Bars: smoothed grid, triangles, halfedges, trimap, mesh normals (before the bilateral)
and FC data bit-identical; bilateral normals within 1e-12 (tests/test_gpu_strict.py);
labels identical; the reference's DegenerateInputError / ValueError cases raise the same
exception types.  Skips when baseline/_ref is absent.
"""

import os
import sys

import numpy as np
import pytest
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")
STUBS = os.path.join(REPO, "tests", "golden", "_stubs")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device"),
              pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "flatpoly")),
                                 reason="baseline/_ref missing (run baseline/install_ref.sh)")]


@pytest.fixture(scope="module")
def ref():
    for p in (STUBS, REF):
        if p not in sys.path:
            sys.path.insert(0, p)
    import flatpoly
    from flatpoly import _kernels, geometry, mesh, segmentation, smoothing
    assert _kernels.ACTIVE == "native", _kernels.ACTIVE     # the compiled reference
    return type("Ref", (), dict(flatpoly=flatpoly, mesh=mesh, smoothing=smoothing,
                                segmentation=segmentation, geometry=geometry))


@pytest.fixture(scope="module")
def fe():
    import paper_2007_12065_b200 as m
    return m


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and \
        np.array_equal(np.isnan(a), np.isnan(b)) and np.array_equal(np.nan_to_num(a), np.nan_to_num(b))


def random_cloud(rng):
    M, N = int(rng.integers(4, 160)), int(rng.integers(4, 160))
    u, v = np.meshgrid(np.arange(M, dtype=float), np.arange(N, dtype=float), indexing="ij")
    s = rng.uniform(0.002, 0.05)
    opc = np.stack([v * s, -u * s, rng.normal(0, 0.01, (M, N)) +
                    0.2 * np.sin(np.arange(N) / rng.uniform(3, 15))[None, :]], axis=2)
    opc += rng.normal(scale=rng.uniform(0, 0.004), size=opc.shape)
    opc += rng.uniform(-5, 5, size=3)                         # away from the origin
    for a, b in rng.integers(0, [M - 1, N - 1], size=(int(rng.integers(0, 6)), 2)):
        opc[a, b + 1] = opc[a, b]                             # coincident vertices
    opc[rng.random((M, N)) < rng.uniform(0, 0.35)] = np.nan
    return opc


@pytest.mark.parametrize("seed", range(24))
def test_drop_in_chain_equals_stock_reference(fe, ref, seed):
    rng = np.random.default_rng(9100 + seed)
    opc = random_cloud(rng)
    M, N = opc.shape[:2]
    k_lap = int(rng.choice([3, 3, 5, 7, 9]))
    if min(M, N) < k_lap:
        k_lap = 3
    lap = (float(rng.uniform(0.2, 1.0)), k_lap, int(rng.integers(1, 6)))
    bil = (float(rng.uniform(0.02, 0.3)), float(rng.uniform(0.05, 0.5)),
           int(rng.choice([3, 3, 5, 7])), int(rng.integers(1, 4)))
    dn = rng.normal(size=(int(rng.integers(1, 6)), 3))
    dn /= np.linalg.norm(dn, axis=1)[:, None]
    l_max, ang_min = float(rng.uniform(0.005, 0.06)), float(rng.uniform(0.7, 0.99))

    r_sm = ref.smoothing.laplacian_filter_opc(opc, ref.smoothing.LaplacianParams(*lap))
    g_sm = fe.laplacian_filter_opc(opc, fe.LaplacianParams(*lap))
    assert same(g_sm, r_sm), seed

    r_mesh = ref.mesh.mesh_from_opc(r_sm)
    g_mesh = fe.mesh_from_opc(g_sm)
    for name in ("triangles", "halfedges", "trimap"):
        assert same(getattr(g_mesh, name), getattr(r_mesh, name)), (seed, name)
    assert same(g_mesh.normals, r_mesh.normals), seed
    r_cen, r_nrm = ref.smoothing.compute_fc_triangle_data(r_sm)
    g_cen, g_nrm = fe.compute_fc_triangle_data(g_sm)
    assert same(g_cen, r_cen) and same(g_nrm, r_nrm), seed

    r_n = ref.smoothing.bilateral_filter_opc(r_sm, ref.smoothing.BilateralParams(*bil),
                                             r_mesh.trimap)
    g_n = fe.bilateral_filter_opc(g_sm, fe.BilateralParams(*bil), g_mesh.trimap)
    assert g_n.shape == r_n.shape and g_n.dtype == r_n.dtype
    bad = np.isnan(r_n).any(1)
    assert np.array_equal(np.isnan(g_n).any(1), bad), seed
    if (~bad).any():
        err = np.linalg.norm(g_n[~bad] - r_n[~bad], axis=1).max()
        assert err <= 1e-12, (seed, err)

    r_mesh.normals, g_mesh.normals = r_n, g_n
    r_lab = ref.segmentation.group_assignment(r_mesh, dn, l_max, ang_min)
    g_lab = fe.group_assignment(g_mesh, dn, l_max, ang_min)
    assert same(g_lab, r_lab), seed


def test_error_types_match_stock_reference(fe, ref):
    """The reference's input errors raise the same exception types from the drop-in."""
    small = np.zeros((2, 2, 3))
    cases = [
        (lambda m: m.smoothing.laplacian_filter_opc(small, m.smoothing.LaplacianParams(1.0, 3, 1)),
         lambda: fe.laplacian_filter_opc(small, fe.LaplacianParams(1.0, 3, 1))),
        (lambda m: m.mesh.mesh_from_opc(np.zeros((1, 5, 3))),
         lambda: fe.mesh_from_opc(np.zeros((1, 5, 3)))),
        (lambda m: m.smoothing.LaplacianParams(1.5, 3, 1), lambda: fe.LaplacianParams(1.5, 3, 1)),
        (lambda m: m.smoothing.BilateralParams(0.1, 0.15, 4, 1),
         lambda: fe.BilateralParams(0.1, 0.15, 4, 1)),
    ]
    opc = np.random.default_rng(1).normal(size=(6, 7, 3))
    bad = np.arange(2 * 5 * 6, dtype=np.int64)
    bad[-1] = 10 ** 9                                       # out-of-range GID entry
    cases.append((lambda m: m.smoothing.bilateral_filter_opc(
        opc, m.smoothing.BilateralParams(0.1, 0.15, 3, 1), bad),
        lambda: fe.bilateral_filter_opc(opc, fe.BilateralParams(0.1, 0.15, 3, 1), bad)))
    for r_call, g_call in cases:
        with pytest.raises(Exception) as r_exc:
            r_call(ref)
        with pytest.raises(Exception) as g_exc:
            g_call()
        assert isinstance(g_exc.value, ValueError) == isinstance(r_exc.value, ValueError)
        assert type(g_exc.value).__name__ == type(r_exc.value).__name__, \
            (type(g_exc.value), type(r_exc.value))


@pytest.mark.parametrize("case", ["lidar_k3", "lidar_k5_13", "room_k11", "lidar_big"])
def test_structured_scenes_equal_stock_reference(fe, ref, case):
    """Range images (the C3 scanner: NaN rows / sky, 80 m ranges) and a room at large
    kernel sizes through the drop-in chain and the stock reference, incl. l_max group
    labels -- same bars as the random clouds."""
    if case.startswith("lidar"):
        rows, cols = (64, 1024) if case == "lidar_big" else (32, 256)
        opc = fe.synthetic.lidar_scan(rows=rows, cols=cols, seed=11)
        lap = {"lidar_k3": (1.0, 3, 5), "lidar_k5_13": (0.6, 5, 3), "lidar_big": (1.0, 3, 5)}[case]
        bil = {"lidar_k3": (0.3, 0.2, 3, 3), "lidar_k5_13": (0.3, 0.2, 13, 2),
               "lidar_big": (0.3, 0.2, 3, 5)}[case]
        l_max = 0.5
    else:
        opc = fe.synthetic.room_scene(n=120, noise=0.002, seed=9)
        lap, bil, l_max = (0.9, 11, 2), (0.1, 0.15, 11, 2), 0.05
    dn = np.array([[0, 0, 1.0], [1.0, 0, 0], [0, 1.0, 0], [-1.0, 0, 0], [0, -1.0, 0]])

    r_sm = ref.smoothing.laplacian_filter_opc(opc, ref.smoothing.LaplacianParams(*lap))
    g_sm = fe.laplacian_filter_opc(opc, fe.LaplacianParams(*lap))
    assert same(g_sm, r_sm)
    r_mesh, g_mesh = ref.mesh.mesh_from_opc(r_sm), fe.mesh_from_opc(g_sm)
    for name in ("triangles", "halfedges", "trimap", "normals"):
        assert same(getattr(g_mesh, name), getattr(r_mesh, name)), name
    r_n = ref.smoothing.bilateral_filter_opc(r_sm, ref.smoothing.BilateralParams(*bil),
                                             r_mesh.trimap)
    g_n = fe.bilateral_filter_opc(g_sm, fe.BilateralParams(*bil), g_mesh.trimap)
    bad = np.isnan(r_n).any(1)
    assert np.array_equal(np.isnan(g_n).any(1), bad)
    assert np.linalg.norm(g_n[~bad] - r_n[~bad], axis=1).max() <= 1e-12
    r_mesh.normals, g_mesh.normals = r_n, g_n
    assert same(fe.group_assignment(g_mesh, dn, l_max, 0.9),
                ref.segmentation.group_assignment(r_mesh, dn, l_max, 0.9))


@pytest.mark.parametrize("seed", range(12))
def test_mixed_front_end_vs_stock_reference(fe, ref, seed):
    """FrontEnd(precision="mixed") on random clouds against the stock reference's chain:
    smoothed grid within 1e-12 relative, topology identical, normals within the 1e-5
    contract."""
    rng = np.random.default_rng(9300 + seed)
    opc = random_cloud(rng)
    M, N = opc.shape[:2]
    lap = (float(rng.uniform(0.2, 1.0)), 3, int(rng.integers(1, 6)))
    bil = (float(rng.uniform(0.02, 0.3)), float(rng.uniform(0.05, 0.5)),
           int(rng.choice([3, 5, 7])), int(rng.integers(1, 4)))
    r_sm = ref.smoothing.laplacian_filter_opc(opc, ref.smoothing.LaplacianParams(*lap))
    r_mesh = ref.mesh.mesh_from_opc(r_sm)
    r_n = ref.smoothing.bilateral_filter_opc(r_sm, ref.smoothing.BilateralParams(*bil),
                                             r_mesh.trimap)
    eng = fe.FrontEnd(M, N, 1, laplacian=fe.LaplacianParams(*lap),
                      bilateral=fe.BilateralParams(*bil), src_dtype=torch.float64,
                      precision="mixed")
    res = eng.run(torch.from_numpy(opc).cuda().unsqueeze(0))
    T = res.n_tri[0]
    pts, ok = res.points[0].cpu().numpy(), np.isfinite(r_sm).all(2)
    assert np.array_equal(np.isnan(pts), np.isnan(r_sm))
    if ok.any():
        rel = np.linalg.norm(pts[ok] - r_sm[ok], axis=1) / np.linalg.norm(r_sm[ok], axis=1)
        assert rel.max() <= 1e-12
    assert np.array_equal(res.trimap[0].cpu().numpy(), r_mesh.trimap)
    assert np.array_equal(res.triangles[0, :T].cpu().numpy(), r_mesh.triangles)
    g_n = res.normals[0, :T].cpu().numpy()
    bad = np.isnan(r_n).any(1)
    assert np.array_equal(np.isnan(g_n).any(1), bad)
    if (~bad).any():
        assert np.linalg.norm(g_n[~bad] - r_n[~bad], axis=1).max() <= 1e-5
