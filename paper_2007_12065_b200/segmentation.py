"""Per-triangle group labels: the data-parallel head of the reference's segmentation.

Reference: flatpoly/segmentation.py:52-74.  ``group_assignment`` labels every triangle
with the index of its best dominant normal (argmax of n . d), UNASSIGNED (255) when the
best score is below ang_min (NaN normals included) or when the longest edge exceeds
l_max (segmentation.py:59-67,73 -- the north-star's "max edge length masking", which
never changes the mesh: validity is NaN-only, mesh.py:81-82).  Both run on the GPU in
fp64: edge lengths bit-exact, scores in the FMA order of numpy's BLAS matmul.

Region growing (segmentation.py:76-170): ``extract_planar_segment``
(one seed, the reference's kernel call) and ``grow_segments`` (every segment of one label,
in region_growing_task's order) on the GPU -- a segment is the connected component of its
seed among the eligible triangles (csrc/segments.cu), so the membership sets are exact.
Plane fitting (np.linalg.eigh) and polygon extraction stay out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _ops
from ._device import Staged, host_view

UNASSIGNED = np.uint8(255)
MAX_GROUPS = 254


def max_edge_mask(mesh, l_max: float):
    """bool per triangle: longest edge > l_max (segmentation.py:59-67,73)."""
    P = Staged(mesh.points)
    tri = Staged(mesh.triangles, float_only=False).dev.to(torch.int64).reshape(-1, 3).contiguous()
    out = _ops.max_edge_mask(P.dev.reshape(-1, 3).contiguous(), tri, l_max)
    return P.give(out)


def group_assignment(mesh, dominant_normals, l_max: float, ang_min: float):
    """Per-triangle group labels (uint8); iteration-order independent (segmentation.py:52-74)."""
    dn = np.atleast_2d(np.asarray(dominant_normals, dtype=np.float64))
    if not 1 <= len(dn) <= MAX_GROUPS:
        raise ValueError(f"need 1..{MAX_GROUPS} dominant normals, got {len(dn)}")
    P = Staged(mesh.points)
    pts = P.dev.reshape(-1, 3).contiguous()
    tri = Staged(mesh.triangles, float_only=False).dev.to(torch.int64).reshape(-1, 3).contiguous()
    nrm = Staged(mesh.normals).dev.reshape(-1, 3).contiguous()
    lflag = _ops.max_edge_mask(pts, tri, l_max).to(torch.uint8)
    labels = _ops.group_assignment(nrm, host_view(dn), ang_min, lflag=lflag)
    return P.give(labels)


@dataclass
class SegmentationParams:
    """segmentation.py:26-39 (same defaults, same validation messages)."""
    l_max: float = 0.1
    ang_min: float = 0.95
    ptp_max: float = 0.0
    tri_min: int = 10
    vertices_hole_min: int = 3

    def __post_init__(self):
        if not 0.0 < self.ang_min <= 1.0:
            raise ValueError("ang_min must be in (0, 1]")
        if self.tri_min < 1:
            raise ValueError("tri_min must be >= 1")
        if self.vertices_hole_min < 3:
            raise ValueError("vertices_hole_min must be >= 3")


def _seed_anchor(points, triangles, seed):
    """The seed triangle's centroid, as segmentation.py:86 computes it (numpy mean)."""
    if isinstance(points, torch.Tensor):  # 9 doubles to the host: the same numpy reduction
        tri = triangles[int(seed)].to(torch.int64)
        return points.reshape(-1, 3)[tri].to(torch.float64).cpu().numpy().mean(axis=0)
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    return pts[np.asarray(triangles)[int(seed)]].mean(axis=0)


def extract_planar_segment(seed: int, mesh, groups, dominant_normal, ptp_max: float, visited):
    """Edge-connected triangles reachable from ``seed`` within its group
    (segmentation.py:76-91); joined triangles are marked in ``visited``."""
    from . import _kernels
    anchor = _seed_anchor(mesh.points, mesh.triangles, seed)
    label = int(groups[int(seed)])
    return _kernels.grow_segment(mesh.triangles, mesh.halfedges, mesh.points, groups, visited,
                                 int(seed), label, anchor,
                                 np.ascontiguousarray(dominant_normal, dtype=np.float64),
                                 float(ptp_max))


def grow_segments(mesh, groups, label: int, dominant_normal, params: SegmentationParams):
    """The ``triangle_indices`` of every segment region_growing_task (segmentation.py:117-151)
    keeps for ``label``, in its order: seeds in ascending index, segments of at least
    ``params.tri_min`` triangles, members sorted.  NumPy mesh -> list of int64 arrays;
    torch (CUDA) mesh -> list of device tensors.

    ptp_max == 0 (the default): one union-find pass gives every component at once (the
    seed of a segment is its minimum index).  ptp_max > 0: the anchor depends on the seed,
    so seeds are taken one at a time, each segment one union-find pass over the eligible
    triangles of that anchor (csrc/segments.cu)."""
    from ._device import Staged
    host = not isinstance(groups, torch.Tensor)
    G = Staged(groups, float_only=False).dev.to(torch.uint8).contiguous()
    HE = Staged(mesh.halfedges, float_only=False).dev.to(torch.int64).contiguous()
    n = int(G.shape[0])
    out = []
    if n == 0:
        return out
    if float(params.ptp_max) <= 0.0:
        comp, size = _ops.segment_components(HE, G)
        lab = G == int(label)
        keep = lab & (comp >= 0)
        keep &= size[comp.clamp(min=0)] >= int(params.tri_min)
        idx = torch.nonzero(keep).flatten()
        roots = comp[idx]
        order = torch.argsort(roots, stable=True)   # groups by root, members ascending
        idx, roots = idx[order], roots[order]
        _, counts = torch.unique_consecutive(roots, return_counts=True)
        parts = torch.split(idx, counts.tolist())
    else:
        T = Staged(mesh.triangles, float_only=False).dev.to(torch.int64).reshape(-1, 3).contiguous()
        P = Staged(mesh.points).dev.to(torch.float64).reshape(-1, 3).contiguous()
        dn = np.ascontiguousarray(dominant_normal, dtype=np.float64)
        visited = torch.zeros((n,), dtype=torch.uint8, device=G.device)
        cand = torch.nonzero(G == int(label)).flatten()
        parts, pos = [], 0
        while pos < cand.numel():
            free = torch.nonzero(visited[cand[pos:]] == 0)
            if free.numel() == 0:
                break
            rel = int(free[0])
            seed = int(cand[pos + rel])
            pos += rel + 1
            anchor = _seed_anchor(P, T, seed)
            m = _ops.grow_segment(T, HE, P, G, visited, seed, int(label), anchor, dn,
                                  float(params.ptp_max))
            if m.numel() >= int(params.tri_min):
                parts.append(m)
    for p in parts:
        out.append(p.cpu().numpy() if host else p)
    return out


def apply_lmax(labels, mask):
    """labels[mask] = UNASSIGNED, as segmentation.py:73 does after the angular test."""
    labels = labels.copy() if isinstance(labels, np.ndarray) else labels.clone()
    labels[mask] = 255
    return labels
