"""Geometry primitives on the hot path (reference: flatpoly/geometry.py).

Only what the OPC front-end needs: the error type (geometry.py:21-22) and the
vectorised triangle normals (geometry.py:134-147), computed on the GPU in fp64
with numpy's operation order, so float64 results are bit-identical.
"""

from __future__ import annotations

import torch

from . import _ops
from ._device import Staged


class DegenerateInputError(ValueError):
    """Input does not carry enough geometry to operate on (geometry.py:21-22)."""


def triangle_normals(points, triangles):
    """Per-triangle unit normals, NaN for degenerate triangles (geometry.py:134-147)."""
    P = Staged(points)
    T = Staged(triangles, float_only=False)
    tri = T.dev.to(dtype=torch.int64).reshape(-1, 3).contiguous()
    pts = P.dev.reshape(-1, 3)
    return P.give(_ops.triangle_normals(pts, tri))
