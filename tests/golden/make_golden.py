"""Generate golden vectors by running the REAL reference (flatpoly) in this container.

    python tests/golden/make_golden.py            # writes tests/golden/*.npz

Needs /root/reference (read-only) and oracle/_ref/_native.so (built from the
reference's own _native.pyx by oracle/build_ref.sh).  Nothing at test or bench
time reads /root/reference: the .npz files produced here are committed.

Reference functions called (paths relative to /root/reference/pkg/src/flatpoly):
  mesh.extract_triangles_opc (mesh.py:58), mesh.extract_halfedges_opc (:99),
  mesh.mesh_from_opc (:167), smoothing.compute_fc_triangle_data (smoothing.py:61),
  smoothing.laplacian_filter_opc (:53), smoothing.bilateral_filter_opc (:91),
  _kernels._fallback.{laplacian_filter, bilateral_iterate} (semantics of record),
  _kernels._native.{laplacian_filter, bilateral_iterate} (compiled backend),
  segmentation.group_assignment (segmentation.py:52), synthetic.room_scene (synthetic.py:42),
  pipeline.run_scene organized branch sequence (pipeline.py:125-134).
"""

from __future__ import annotations

import importlib.util
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"


def load_reference():
    sys.path.insert(0, os.path.join(HERE, "_stubs"))      # shapely import stub
    sys.path.insert(0, REF_SRC)
    so = os.path.join(REPO, "oracle", "_ref", "_native.so")
    spec = importlib.util.spec_from_file_location("flatpoly._kernels._native", so)
    native = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(native)
    sys.modules["flatpoly._kernels._native"] = native      # so _kernels picks "native"
    import flatpoly  # noqa: F401
    from flatpoly import _kernels
    assert _kernels.ACTIVE == "native", _kernels.ACTIVE
    return native


def grid_opc(M, N, z=0.0):
    u, v = np.meshgrid(np.arange(M, dtype=float), np.arange(N, dtype=float), indexing="ij")
    return np.stack([v, -u, np.full_like(u, z)], axis=2)


def lidar_scan(rows=16, cols=128, seed=3):
    """Small spinning-LiDAR range image with NaN gaps (SURVEY Appendix B, C3 recipe)."""
    rng = np.random.default_rng(seed)
    el = np.deg2rad(np.linspace(15.0, -25.0, rows))[:, None]
    az = np.linspace(-np.pi, np.pi, cols, endpoint=False)[None, :]
    d = np.stack([np.cos(el) * np.cos(az), np.cos(el) * np.sin(az),
                  np.sin(el) * np.ones_like(az)], axis=2)
    o = np.array([0.0, 0.0, 1.73])
    best = np.full((rows, cols), np.inf)
    with np.errstate(divide="ignore", invalid="ignore"):
        t = (0.0 - o[2]) / d[..., 2]
        best = np.where((t > 0) & (t < best), t, best)
        for axis, c in ((0, 15.0), (0, -15.0), (1, 8.0), (1, -8.0)):
            t = (c - o[axis]) / d[..., axis]
            z = o[2] + t * d[..., 2]
            ok = (t > 0) & (z >= 0) & (z <= 3.0) & (t < best)
            best = np.where(ok, t, best)
    best = best + rng.normal(0.0, 0.01, best.shape)
    best[(best > 80) | ~np.isfinite(best)] = np.nan
    best[rng.random(best.shape) < 0.03] = np.nan
    return o + best[..., None] * d


def main():
    native = load_reference()
    from flatpoly._kernels import _fallback
    from flatpoly.mesh import extract_halfedges_opc, extract_triangles_opc, mesh_from_opc
    from flatpoly.segmentation import group_assignment
    from flatpoly.smoothing import (BilateralParams, LaplacianParams, bilateral_filter_opc,
                                    compute_fc_triangle_data, laplacian_filter_opc)
    from flatpoly.synthetic import flat_plane_opc, room_scene

    # ---------------------------------------------------------------- topology
    topo = {}
    rng = np.random.default_rng(12345)
    cases = [("quad2x2", grid_opc(2, 2)), ("grid2x3", grid_opc(2, 3))]
    o = grid_opc(2, 2)
    o[0, 1] = np.nan
    cases.append(("quad2x2_p2nan", o))
    o = grid_opc(7, 7)
    o[rng.random((7, 7)) < 0.3] = np.nan
    cases.append(("nan7x7", o))
    for i in range(24):
        M = int(rng.integers(2, 14))
        N = int(rng.integers(2, 14))
        o = grid_opc(M, N)
        o[..., 2] = rng.normal(0, 0.1, (M, N))
        o[rng.random((M, N)) < rng.uniform(0, 0.6)] = np.nan
        cases.append((f"rand{i:02d}", o))
    for name, (M, N, dens) in {"big37x53": (37, 53, 0.4), "big64x33": (64, 33, 0.05)}.items():
        o = grid_opc(M, N)
        o[..., 2] = rng.normal(0, 0.1, (M, N))
        o[rng.random((M, N)) < dens] = np.nan
        cases.append((name, o))
    for name, opc in cases:
        tris, trimap = extract_triangles_opc(opc)
        he = extract_halfedges_opc(trimap, opc.shape[0], opc.shape[1])
        mesh = mesh_from_opc(opc)
        assert np.array_equal(mesh.triangles, tris) and np.array_equal(mesh.halfedges, he)
        cen, nrm = compute_fc_triangle_data(opc)
        topo[f"{name}/opc"] = opc
        topo[f"{name}/triangles"] = tris
        topo[f"{name}/trimap"] = trimap
        topo[f"{name}/halfedges"] = he
        topo[f"{name}/normals"] = mesh.normals
        topo[f"{name}/fc_centroids"] = cen
        topo[f"{name}/fc_normals"] = nrm
    np.savez_compressed(os.path.join(HERE, "topology.npz"), **topo)

    # --------------------------------------------------------------- laplacian
    lap = {}
    rng = np.random.default_rng(2024)
    o = flat_plane_opc(12, 9, spacing=0.1, noise=0.01, seed=3)
    lap["border/opc"] = o
    lap["border/params"] = np.array([0.8, 3, 4])
    lap["border/out"] = laplacian_filter_opc(o, LaplacianParams(lam=0.8, kernel_size=3, iterations=4))
    o = flat_plane_opc(20, 30, spacing=0.05, noise=0.01, seed=4)
    o[rng.random((20, 30)) < 0.15] = np.nan
    for k in (3, 5, 7):
        lap[f"nan_k{k}/opc"] = o
        lap[f"nan_k{k}/params"] = np.array([0.8, k, 3])
        lap[f"nan_k{k}/out"] = _fallback.laplacian_filter(o, 0.8, k, 3)
        lap[f"nan_k{k}/out_native"] = native.laplacian_filter(o, 0.8, k, 3)
    o = flat_plane_opc(7, 7, spacing=1.0)
    o[3, 3, 2] = 0.5
    lap["displaced/opc"] = o
    lap["displaced/params"] = np.array([1.0, 3, 1])
    lap["displaced/out"] = laplacian_filter_opc(o, LaplacianParams(lam=1.0, kernel_size=3, iterations=1))
    o = np.full((5, 5, 3), np.nan)
    lap["allnan/opc"] = o
    lap["allnan/params"] = np.array([1.0, 3, 1])
    lap["allnan/out"] = laplacian_filter_opc(o, LaplacianParams())
    o = flat_plane_opc(33, 41, spacing=0.02, noise=0.003, seed=8)
    o[rng.random((33, 41)) < 0.05] = np.nan
    o[5, 7, 1] = np.nan                           # partial-NaN vertex
    lap["partial/opc"] = o
    lap["partial/params"] = np.array([0.6, 3, 10])
    lap["partial/out"] = laplacian_filter_opc(o, LaplacianParams(lam=0.6, kernel_size=3, iterations=10))
    np.savez_compressed(os.path.join(HERE, "laplacian.npz"), **lap)

    # --------------------------------------------------------------- bilateral
    bil = {}
    rng = np.random.default_rng(777)
    o = flat_plane_opc(18, 22, spacing=0.05, noise=0.01, seed=5)
    o[rng.random((18, 22)) < 0.1] = np.nan
    cen, nrm = compute_fc_triangle_data(o)
    for k, it in ((3, 2), (5, 1)):
        bil[f"iter_k{k}/centroids"] = cen
        bil[f"iter_k{k}/normals"] = nrm
        bil[f"iter_k{k}/params"] = np.array([0.1, 0.15, k, it])
        bil[f"iter_k{k}/out"] = _fallback.bilateral_iterate(cen, nrm, 0.1, 0.15, k, it)
        bil[f"iter_k{k}/out_native"] = native.bilateral_iterate(cen, nrm, 0.1, 0.15, k, it)
    n = 11
    o = np.zeros((n, n, 3))
    for u in range(n):
        for v in range(n):
            x = float(v)
            o[u, v] = [x, -float(u), 0.0] if x <= 5.0 else [5.0, -float(u), -(x - 5.0)]
    o *= 0.05
    bil["rightangle/opc"] = o
    bil["rightangle/params"] = np.array([1.0, 0.1, 3, 1])
    bil["rightangle/out"] = bilateral_filter_opc(o, BilateralParams(sigma_length=1.0, sigma_angle=0.1))
    o = flat_plane_opc(10, 10, spacing=0.05, noise=0.01, seed=4)
    o[rng.random((10, 10)) < 0.15] = np.nan
    bil["nan10/opc"] = o
    bil["nan10/params"] = np.array([0.1, 0.15, 3, 2])
    bil["nan10/out"] = bilateral_filter_opc(o, BilateralParams(iterations=2))
    o = np.full((2, 2, 3), np.nan)
    o[0, 0] = [0, 0, 0]
    o[0, 1] = [1, 0, 0]
    o[1, 1] = [1, -1, 0]
    bil["single/opc"] = o
    bil["single/params"] = np.array([0.1, 0.15, 3, 1])
    bil["single/out"] = bilateral_filter_opc(o, BilateralParams())
    np.savez_compressed(os.path.join(HERE, "bilateral.npz"), **bil)

    # ------------------------------------------------ front end (pipeline.py:125-134)
    fe = {}
    up = np.array([[0.0, 0.0, 1.0]])
    scene = room_scene(n=48, noise=0.002, seed=11)
    lp = LaplacianParams(lam=1.0, kernel_size=3, iterations=2)
    bp = BilateralParams(sigma_length=0.1, sigma_angle=0.15, kernel_size=3, iterations=2)
    sm = laplacian_filter_opc(scene.opc, lp)
    mesh = mesh_from_opc(sm)
    plain_normals = mesh.normals.copy()
    mesh.normals = bilateral_filter_opc(sm, bp, mesh.trimap)
    fe["room/opc"] = scene.opc
    fe["room/lap"] = np.array([1.0, 3, 2])
    fe["room/bil"] = np.array([0.1, 0.15, 3, 2])
    fe["room/smoothed"] = sm
    fe["room/triangles"] = mesh.triangles
    fe["room/trimap"] = mesh.trimap
    fe["room/halfedges"] = mesh.halfedges
    fe["room/mesh_normals"] = plain_normals
    fe["room/normals"] = mesh.normals
    # l_max: group labels with the angular filter disabled vs enabled on l_max
    for l_max in (0.05, 0.5):
        lab = group_assignment(mesh, up, l_max, 1e-12)
        lab_inf = group_assignment(mesh, up, np.inf, 1e-12)
        fe[f"room/labels_lmax{l_max}"] = lab
        fe[f"room/labels_lmaxinf"] = lab_inf
    # LiDAR-like range image: 5 Laplacian iterations + l_max mask (config C3 recipe)
    o = lidar_scan()
    sm = laplacian_filter_opc(o, LaplacianParams(lam=1.0, kernel_size=3, iterations=5))
    mesh = mesh_from_opc(sm)
    fe["lidar/opc"] = o
    fe["lidar/lap"] = np.array([1.0, 3, 5])
    fe["lidar/smoothed"] = sm
    fe["lidar/triangles"] = mesh.triangles
    fe["lidar/trimap"] = mesh.trimap
    fe["lidar/halfedges"] = mesh.halfedges
    fe["lidar/mesh_normals"] = mesh.normals
    # normals pointing every way: use both +z and -z... compare only triangles the
    # angular filter keeps (labels_lmaxinf != 255)
    dn = np.array([[0.0, 0.0, 1.0], [0.0, 0.0, -1.0], [1.0, 0, 0], [-1.0, 0, 0],
                   [0, 1.0, 0], [0, -1.0, 0]])
    fe["lidar/labels_lmax0.5"] = group_assignment(mesh, dn, 0.5, 1e-12)
    fe["lidar/labels_lmaxinf"] = group_assignment(mesh, dn, np.inf, 1e-12)
    # known answer (tests/test_segmentation.py:20-26): 3x3 grid, spacing 1
    mesh = mesh_from_opc(flat_plane_opc(3, 3, spacing=1.0))
    fe["grid3/opc"] = flat_plane_opc(3, 3, spacing=1.0)
    fe["grid3/labels_lmax0.5"] = group_assignment(mesh, up, 0.5, 0.5)
    fe["grid3/labels_lmax2.0"] = group_assignment(mesh, up, 2.0, 0.5)
    np.savez_compressed(os.path.join(HERE, "frontend.npz"), **fe)

    # ------------------------------------------------- group_assignment (segmentation.py:52)
    grp = {}
    from flatpoly.mesh import HalfEdgeMesh
    planes = np.array([[0, 0, 1.0], [-1.0, 0, 0], [1.0, 0, 0], [0, -1.0, 0], [0, 1.0, 0]])
    sm = laplacian_filter_opc(scene.opc, lp)
    mesh = mesh_from_opc(sm)
    mesh.normals = bilateral_filter_opc(sm, bp, mesh.trimap)
    for name, (msh, dn, l_max, ang) in {
            "room": (mesh, planes, 0.5, 0.96),
            "room_loose": (mesh, planes[:3], 0.5, 0.5)}.items():
        grp[f"{name}/points"] = msh.points
        grp[f"{name}/triangles"] = msh.triangles
        grp[f"{name}/normals"] = msh.normals
        grp[f"{name}/dominant"] = dn
        grp[f"{name}/params"] = np.array([l_max, ang])
        grp[f"{name}/labels"] = group_assignment(msh, dn, l_max, ang)
    rng = np.random.default_rng(99)
    pts = rng.normal(size=(3000, 3))
    tris = rng.integers(0, 3000, size=(6000, 3))
    nrm = rng.normal(size=(6000, 3))
    nrm /= np.linalg.norm(nrm, axis=1)[:, None]
    nrm[rng.random(6000) < 0.05] = np.nan
    dn = rng.normal(size=(40, 3))
    dn /= np.linalg.norm(dn, axis=1)[:, None]
    msh = HalfEdgeMesh(points=pts, triangles=tris, halfedges=None, normals=nrm)
    grp["random/points"], grp["random/triangles"], grp["random/normals"] = pts, tris, nrm
    grp["random/dominant"] = dn
    grp["random/params"] = np.array([3.0, 0.6])
    grp["random/labels"] = group_assignment(msh, dn, 3.0, 0.6)
    # exact normal match at ang_min = 1.0 (tests/test_segmentation.py:28-31)
    msh = mesh_from_opc(flat_plane_opc(3, 3, spacing=0.1))
    grp["exact/points"], grp["exact/triangles"], grp["exact/normals"] = \
        msh.points, msh.triangles, msh.normals
    grp["exact/dominant"] = up
    grp["exact/params"] = np.array([1.0, 1.0])
    grp["exact/labels"] = group_assignment(msh, up, 1.0, 1.0)
    np.savez_compressed(os.path.join(HERE, "groups.npz"), **grp)

    # ------------------------------------ FastGA cell search (_kernels.find_cells, 8f rank 2)
    from flatpoly import sfc
    from flatpoly.accumulator import build_accumulator, integrate_normals
    ga_out = {}
    rng = np.random.default_rng(4242)
    for level in (2, 4):
        ga = build_accumulator(level)
        q = rng.normal(size=(20000, 3))
        q /= np.linalg.norm(q, axis=1)[:, None]
        q[:50] *= 3.7                               # non-unit rows (normalised inside s2_id)
        q[50:60] = ga.normals[:10]                  # exact cell normals
        args = (q, ga.s2ids, ga.normals, ga.neighbors, ga.model_slope, ga.model_intercept,
                ga.window_lo, ga.window_hi)
        key = f"level{level}"
        ga_out[f"{key}/queries"] = q
        ga_out[f"{key}/ids"] = ga.s2ids
        ga_out[f"{key}/cell_normals"] = ga.normals
        ga_out[f"{key}/neighbors"] = ga.neighbors
        ga_out[f"{key}/model"] = np.array([ga.model_slope, ga.model_intercept,
                                            ga.window_lo, ga.window_hi])
        ga_out[f"{key}/s2id"] = sfc.s2_id(q)
        ga_out[f"{key}/cells"] = _fallback.find_cells(*args)
        ga_out[f"{key}/cells_native"] = native.find_cells(*args)
        # integrate_normals over the room mesh normals (bilateral), 12 % sampling
        ga.counts[:] = 0
        counts = integrate_normals(ga, mesh.normals, sample_pct=0.12)
        ga_out[f"{key}/mesh_normals"] = mesh.normals
        ga_out[f"{key}/counts"] = counts.copy()
    np.savez_compressed(os.path.join(HERE, "fastga.npz"), **ga_out)
    for f in ("topology", "laplacian", "bilateral", "frontend", "groups", "fastga"):
        p = os.path.join(HERE, f + ".npz")
        print(f"{p}: {os.path.getsize(p) / 1024:.1f} KiB")


if __name__ == "__main__":
    main()
