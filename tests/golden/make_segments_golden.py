"""Region-growing golden vectors from the REAL reference.

    python tests/golden/make_segments_golden.py     # writes tests/golden/segments.npz

Two noisy room scenes (4 % and 25 % dropout: one large segment per wall, and many small
fragments around tri_min) are meshed by the reference (mesh.mesh_from_opc),
labelled by segmentation.group_assignment against the 6 axis normals, and every label is
grown by segmentation.region_growing_task (segmentation.py:117-170; native grow_segment
backend, _native.pyx:170-222) with the planarity check off (ptp_max = 0, the default)
and on (ptp_max = 0.01 m).  Recorded: the mesh, the labels, and each run's segments'
triangle_indices (concatenated + lengths).  Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import load_reference  # noqa: E402

DN = np.array([[0, 0, 1.0], [0, 0, -1.0], [1.0, 0, 0], [-1.0, 0, 0], [0, 1.0, 0], [0, -1.0, 0]])


def main():
    load_reference()
    from flatpoly import mesh as rmesh
    from flatpoly import segmentation as rseg
    from flatpoly import synthetic as rsyn
    from flatpoly._kernels import ACTIVE

    assert ACTIVE == "native"
    out = dict(dominant=DN)
    # (scene n, range noise, dropout, tri_min): a clean room and a fragmented one
    for name, n, noise, drop, tri_min in (("room", 120, 0.004, 0.04, 10),
                                          ("frag", 90, 0.006, 0.25, 3)):
        scene = rsyn.room_scene(n=n, noise=noise, seed=5)
        opc = np.array(scene.opc, dtype=np.float64)
        opc[np.random.default_rng(55).random(opc.shape[:2]) < drop] = np.nan
        mesh = rmesh.mesh_from_opc(opc)
        groups = rseg.group_assignment(mesh, DN, l_max=0.08, ang_min=0.9)
        out.update({f"{name}_points": mesh.points, f"{name}_triangles": mesh.triangles,
                    f"{name}_halfedges": mesh.halfedges, f"{name}_groups": groups,
                    f"{name}_tri_min": np.int64(tri_min)})
        for ptp in (0.0, 0.01):
            params = rseg.SegmentationParams(l_max=0.08, ang_min=0.9, ptp_max=ptp,
                                             tri_min=tri_min)
            for lab in range(len(DN)):
                segs, _, _ = rseg.region_growing_task(mesh, groups, lab, DN[lab], params)
                key = f"{name}_ptp{ptp:g}_label{lab}"
                idx = [s.triangle_indices for s in segs]
                out[key + "_members"] = np.concatenate(idx) if idx else np.zeros(0, np.int64)
                out[key + "_lengths"] = np.array([len(i) for i in idx], dtype=np.int64)
                print(key, len(segs), "segments", int(out[key + "_lengths"].sum()), "triangles")
    np.savez_compressed(os.path.join(HERE, "segments.npz"), **out)


if __name__ == "__main__":
    main()
