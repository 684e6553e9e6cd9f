"""Per-triangle group labels: the data-parallel head of the reference's segmentation.

Reference: flatpoly/segmentation.py:52-74.  ``group_assignment`` labels every triangle
with the index of its best dominant normal (argmax of n . d), UNASSIGNED (255) when the
best score is below ang_min (NaN normals included) or when the longest edge exceeds
l_max (segmentation.py:59-67,73 -- the north-star's "max edge length masking", which
never changes the mesh: validity is NaN-only, mesh.py:81-82).  Both run on the GPU in
fp64: edge lengths bit-exact, scores in the FMA order of numpy's BLAS matmul.  Region
growing / plane fitting (segmentation.py:77-170) are outside this build's hot path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _ops
from ._device import Staged

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
    labels = _ops.group_assignment(nrm, torch.from_numpy(dn), ang_min, lflag=lflag)
    return P.give(labels)


def apply_lmax(labels, mask):
    """labels[mask] = UNASSIGNED, as segmentation.py:73 does after the angular test."""
    labels = labels.copy() if isinstance(labels, np.ndarray) else labels.clone()
    labels[mask] = 255
    return labels
