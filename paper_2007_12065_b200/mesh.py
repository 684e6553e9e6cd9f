"""OPC mesh front-end (reference: flatpoly/mesh.py, OPC part).

Implicit right-cut triangulation of an organized (M, N, 3) cloud with the GID
map and twin half-edges, computed by one sm_100a kernel pass
(libopcfe ``opcfe_triangulate``).  Same names, arguments, conventions and
errors as the reference:

* GID = 2*(u*(N-1)+v)+k (mesh.py:46-55);
* triangle t owns half-edges 3t..3t+2, half-edge 3t+k runs from
  triangles[t][k] to triangles[t][(k+1)%3], halfedges[e] is its twin or -1
  (mesh.py:8-10);
* triangles/trimap/halfedges are int64 and bit-identical to the reference;
  normals are float64 and bit-identical for float64 input.

NumPy inputs return NumPy outputs (host); torch CUDA tensors stay on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _ops
from ._device import Staged
from .geometry import DegenerateInputError


@dataclass
class HalfEdgeMesh:
    """Same fields as flatpoly.mesh.HalfEdgeMesh (mesh.py:24-35)."""
    points: object              # (n, 3) float64 -- a view of the caller's grid
    triangles: object           # (t, 3) int64
    halfedges: object           # (3t,) int64, -1 = border
    normals: object = None      # (t, 3) unit normals, NaN when degenerate
    trimap: object = None       # GID -> triangle index (-1 = absent)
    grid_shape: tuple = None    # (M, N)

    @property
    def num_triangles(self) -> int:
        return len(self.triangles)


def edge_origin(mesh: HalfEdgeMesh, e: int) -> int:
    return int(mesh.triangles[e // 3, e % 3])


def edge_dest(mesh: HalfEdgeMesh, e: int) -> int:
    return int(mesh.triangles[e // 3, (e + 1) % 3])


def gid_of(u: int, v: int, k: int, N: int) -> int:
    """Global id of fully-connected triangle (u, v, k) in an M x N grid (mesh.py:46-48)."""
    return 2 * (u * (N - 1) + v) + k


def gid_to_uvk(gid: int, N: int) -> tuple[int, int, int]:
    """Inverse of :func:`gid_of` (mesh.py:51-55)."""
    k = gid & 1
    q = gid >> 1
    return q // (N - 1), q % (N - 1), k


def _check_opc(S: Staged):
    x = S.dev
    if x.dim() != 3 or x.shape[0] < 2 or x.shape[1] < 2 or x.shape[2] != 3:
        raise DegenerateInputError("organized cloud must be at least 2 x 2")
    return x.shape[0], x.shape[1]


def _triangulate(S: Staged, halfedges: bool):
    M, N = _check_opc(S)
    _, vmask = _ops.stage_in(S.dev, want_points=False, want_mask=True)
    r = _ops.triangulate(vmask, 1, M, N, halfedges=halfedges)
    T = int(r["n_tri"][0].item())                     # data-dependent size: one readback
    return M, N, T, r


def extract_triangles_opc(opc):
    """Right-cut triangles of an organized (M, N, 3) cloud plus the GID map (mesh.py:58-96)."""
    S = Staged(opc)
    M, N, T, r = _triangulate(S, halfedges=False)
    return S.give(r["triangles"][0, :T]), S.give(r["trimap"][0])


def extract_halfedges_opc(trimap, M: int, N: int):
    """Twin-edge array for the right-cut OPC triangulation (mesh.py:99-135)."""
    S = Staged(trimap, float_only=False)
    tm = S.dev.to(torch.int64).reshape(-1).contiguous()
    if tm.numel() != 2 * (M - 1) * (N - 1):
        raise DegenerateInputError("trimap does not match the grid shape")
    n_tri = int(tm.max().item()) + 1 if tm.numel() else 0
    return S.give(_ops.halfedges_from_trimap(tm, M, N, n_tri))


def compute_normals(mesh: HalfEdgeMesh):
    """Per-triangle unit normals (NaN for degenerate triangles) (mesh.py:162-164)."""
    from .geometry import triangle_normals
    return triangle_normals(mesh.points, mesh.triangles)


def mesh_from_opc(opc) -> HalfEdgeMesh:
    """Organized cloud -> half-edge mesh with normals and GID map (mesh.py:167-180).

    One triangulation pass emits triangles, trimap and twins; normals are computed
    in fp64 from the caller's own vertices (bit-identical for float64 input).
    """
    S = Staged(opc)
    M, N, T, r = _triangulate(S, halfedges=True)
    tris = r["triangles"][0, :T]
    pts_dev = S.dev.reshape(-1, 3)
    normals = _ops.triangle_normals(pts_dev, tris)
    if S.numpy:
        points = np.asarray(opc, dtype=np.float64).reshape(-1, 3)   # view, as mesh.py:173
    else:
        points = opc.reshape(-1, 3)
    return HalfEdgeMesh(
        points=points,
        triangles=S.give(tris),
        halfedges=S.give(r["halfedges"][0, :3 * T]),
        normals=S.give(normals),
        trimap=S.give(r["trimap"][0]),
        grid_shape=(M, N),
    )


# north-star name (Polylidar3D's pybind API)
extract_tri_mesh_from_organized_point_cloud = mesh_from_opc
