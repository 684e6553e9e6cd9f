"""The l_max ("max edge length") mask of the reference's group assignment.

Reference: flatpoly/segmentation.py:52-74.  ``group_assignment`` labels a
triangle UNASSIGNED (255) when its longest edge exceeds l_max
(segmentation.py:59-67,73) -- the north-star's "max edge length masking".  It
does not change the mesh (triangle validity is NaN-only, mesh.py:81-82), so it is
a separate per-triangle output here, computed in fp64 on the GPU (bit-exact).
The rest of group_assignment (argmax over dominant normals) and region growing
are outside this build's hot path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _ops
from ._device import Staged

UNASSIGNED = np.uint8(255)


def max_edge_mask(mesh, l_max: float):
    """bool per triangle: longest edge > l_max (segmentation.py:59-67,73)."""
    P = Staged(mesh.points)
    tri = Staged(mesh.triangles, float_only=False).dev.to(torch.int64).reshape(-1, 3).contiguous()
    out = _ops.max_edge_mask(P.dev.reshape(-1, 3).contiguous(), tri, l_max)
    return P.give(out)


def apply_lmax(labels, mask):
    """labels[mask] = UNASSIGNED, as segmentation.py:73 does after the angular test."""
    labels = labels.copy() if isinstance(labels, np.ndarray) else labels.clone()
    labels[mask] = 255
    return labels
