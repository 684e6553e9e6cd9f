"""Golden CHAINS: the reference's own organized pipeline, end to end, in fp64.

    python tests/golden/make_chain_golden.py        # writes tests/golden/chain.npz

Runs the REAL reference (flatpoly from /root/reference + its compiled Cython kernels
oracle/_ref/_native.so, see make_golden.py) through the organized branch of
pipeline.run_scene (pipeline.py:125-134):

    sm   = smoothing.laplacian_filter_opc(opc, LaplacianParams)      (smoothing.py:53)
    mesh = mesh.mesh_from_opc(sm)                                     (mesh.py:167)
    mesh.normals = smoothing.bilateral_filter_opc(sm, BilateralParams, mesh.trimap)
    labels = segmentation.group_assignment(mesh, dn, l_max, ang_min)  (segmentation.py:52)

and stores every stage, so the GPU chains (strict and fast) are compared with the
reference's chained result -- not with per-stage restatements fed GPU intermediates.
The l_max flag is segmentation.py:59-67,73's `edge_max > l_max` on the reference mesh.
Nothing at test time reads /root/reference: chain.npz is committed.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import lidar_scan, load_reference  # noqa: E402

AXES = np.array([[0.0, 0.0, 1.0], [0.0, 0.0, -1.0], [1.0, 0, 0], [-1.0, 0, 0], [0, 1.0, 0],
                 [0, -1.0, 0]])
PLANES = np.array([[0, 0, 1.0], [-1.0, 0, 0], [1.0, 0, 0], [0, -1.0, 0], [0, 1.0, 0]])


def cases():
    from flatpoly.synthetic import room_scene
    out = []
    out.append(("room72", room_scene(n=72, noise=0.002, seed=5).opc, (1.0, 3, 3),
                (0.1, 0.15, 3, 3), 0.5, PLANES, 0.96))
    # C2 recipe scaled down: central crop + 2 % i.i.d. dropout
    o = room_scene(n=128, noise=0.002, seed=2).opc[16:112, :].copy()
    o[np.random.default_rng(1000).random(o.shape[:2]) < 0.02] = np.nan
    out.append(("c2crop", o, (1.0, 3, 3), (0.1, 0.15, 3, 2), None, PLANES, 0.9))
    # C3 recipe at 32 x 256: NaN gaps, l_max mask, no bilateral
    out.append(("lidar", lidar_scan(32, 256, seed=3), (1.0, 3, 5), None, 0.5, AXES, 0.9))
    out.append(("lidar_bil", lidar_scan(32, 256, seed=4), (1.0, 3, 2), (0.3, 0.2, 3, 2), 0.5,
                AXES, 0.9))
    # kernel sizes beyond the fp32 kernels' compiled set (generic-window kernels)
    out.append(("k11", room_scene(n=48, noise=0.002, seed=7).opc, (0.8, 11, 2),
                (0.1, 0.15, 11, 2), None, PLANES, 0.9))
    out.append(("k19", room_scene(n=48, noise=0.003, seed=8).opc, (1.0, 19, 1),
                (0.2, 0.3, 19, 1), None, PLANES, 0.9))
    # far from the coordinate origin, small sigma_length (fp32 cancellation stress)
    o = room_scene(n=48, noise=0.002, seed=9).opc + np.array([300.0, -200.0, 50.0])
    out.append(("far", o, (1.0, 3, 2), (0.05, 0.15, 3, 2), None, PLANES, 0.9))
    return out


def main():
    load_reference()
    from flatpoly.mesh import mesh_from_opc
    from flatpoly.segmentation import group_assignment
    from flatpoly.smoothing import (BilateralParams, LaplacianParams, bilateral_filter_opc,
                                    laplacian_filter_opc)
    g = {}
    for name, opc, lap, bil, l_max, dn, ang in cases():
        sm = laplacian_filter_opc(opc, LaplacianParams(*lap))
        mesh = mesh_from_opc(sm)
        if bil is not None:
            mesh.normals = bilateral_filter_opc(sm, BilateralParams(*bil), mesh.trimap)
        g[f"{name}/opc"] = opc
        g[f"{name}/lap"] = np.array(lap, dtype=np.float64)
        g[f"{name}/bil"] = np.array(bil if bil is not None else [], dtype=np.float64)
        g[f"{name}/smoothed"] = sm
        # triangles / twins follow from trimap (and are bit-exact-tested elsewhere);
        # trimap as int32 keeps the fixture small
        assert mesh.trimap.max() < 2 ** 31
        g[f"{name}/trimap"] = mesh.trimap.astype(np.int32)
        g[f"{name}/n_halfedges_linked"] = np.array([(mesh.halfedges >= 0).sum()])
        g[f"{name}/normals"] = mesh.normals
        g[f"{name}/dominant"] = dn
        g[f"{name}/seg"] = np.array([np.inf if l_max is None else l_max, ang])
        g[f"{name}/labels"] = group_assignment(mesh, dn, np.inf if l_max is None else l_max, ang)
        if l_max is not None:
            p, t = mesh.points, mesh.triangles
            a, b, c = p[t[:, 0]], p[t[:, 1]], p[t[:, 2]]
            edge_max = np.maximum(np.linalg.norm(b - a, axis=1),
                                  np.maximum(np.linalg.norm(c - b, axis=1),
                                             np.linalg.norm(a - c, axis=1)))
            g[f"{name}/lmax_flag"] = edge_max > l_max
        print(f"{name}: {opc.shape[:2]} T={mesh.num_triangles}")
    path = os.path.join(HERE, "chain.npz")
    np.savez_compressed(path, **g)
    print(f"{path}: {os.path.getsize(path) / 1024:.1f} KiB")


if __name__ == "__main__":
    main()
