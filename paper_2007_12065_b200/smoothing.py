"""Organized-cloud denoising (reference: flatpoly/smoothing.py).

Laplacian vertex smoothing and bilateral normal smoothing on the image-space
grid, as sm_100a kernels behind libopcfe.  Same dataclasses, validation,
function names and errors as the reference (smoothing.py:22-114).

Precision (north-star contract): arithmetic is fp32 with the fp64 steps the
contract needs (FC normal edges/cross products, l_max edge lengths).  For
float64 input the outputs are float64; vertices / normals the filters leave
unchanged (outer ring, NaN and isolated vertices, unchanged normals) come back
bit-identical, moved ones are within 1e-5 (norm-wise relative) of the fp64
reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _ops
from ._device import Staged
from .geometry import DegenerateInputError


@dataclass
class LaplacianParams:
    """smoothing.py:22-34."""
    lam: float = 1.0
    kernel_size: int = 3
    iterations: int = 1

    def __post_init__(self):
        if not 0.0 < self.lam <= 1.0:
            raise ValueError("lambda must be in (0, 1]")
        if self.kernel_size < 3 or self.kernel_size % 2 == 0:
            raise ValueError("kernel_size must be odd and >= 3")
        if self.iterations < 1:
            raise ValueError("iterations must be >= 1")


@dataclass
class BilateralParams:
    """smoothing.py:37-50."""
    sigma_length: float = 0.1
    sigma_angle: float = 0.15
    kernel_size: int = 3
    iterations: int = 1

    def __post_init__(self):
        if self.sigma_length <= 0 or self.sigma_angle <= 0:
            raise ValueError("sigma scales must be positive")
        if self.kernel_size < 3 or self.kernel_size % 2 == 0:
            raise ValueError("kernel_size must be odd and >= 3")
        if self.iterations < 1:
            raise ValueError("iterations must be >= 1")


def _laplacian_staged(S: Staged, lam, kernel_size, iterations):
    x = S.dev
    M, N = x.shape[:2]
    grid, _ = _ops.stage_in(x, want_points=True, want_mask=False)
    out = _ops.laplacian(grid, 1, M, N, lam, kernel_size, iterations)
    res = _ops.unstage(out, 1, M, N, x.dtype, orig=x.unsqueeze(0))[0]
    return S.give(res)


def laplacian_filter_opc(opc, params: LaplacianParams):
    """Smooth an (M, N, 3) organized cloud; border ring and NaNs are untouched (smoothing.py:53-58)."""
    S = Staged(opc)
    x = S.dev
    if x.dim() != 3 or min(x.shape[:2]) < params.kernel_size:
        raise DegenerateInputError("grid smaller than the filter kernel")
    return _laplacian_staged(S, params.lam, params.kernel_size, params.iterations)


def compute_fc_triangle_data(opc):
    """Centroids and unit normals of the fully-connected triangle grid (smoothing.py:61-88).

    fp64 input -> bit-identical fp64 output (numpy operation order on the GPU).
    """
    S = Staged(opc)
    x = S.dev
    if x.dim() != 3 or x.shape[0] < 2 or x.shape[1] < 2:
        raise DegenerateInputError("organized cloud must be at least 2 x 2")
    cen, nrm = _ops.fc_data(x)
    return S.give(cen), S.give(nrm)


def bilateral_filter_opc(opc, params: BilateralParams, trimap=None):
    """Bilaterally smoothed unit normals for the valid mesh of an OPC (smoothing.py:91-114).

    FC centroids/normals are computed in fp64 from the caller's vertices and
    filtered in fp32; the last pass scatters straight into mesh order through
    the GID map (given, or computed by the triangulation kernel).
    """
    S = Staged(opc)
    x = S.dev
    if x.dim() != 3 or min(x.shape[:2]) < 2:
        raise DegenerateInputError("organized cloud must be at least 2 x 2")
    M, N = x.shape[:2]
    cen, nrm = _ops.fc_data(x)
    if trimap is None:
        _, vmask = _ops.stage_in(x, want_points=False, want_mask=True)
        r = _ops.triangulate(vmask, 1, M, N, halfedges=False)
        tm = r["trimap"][0]
    else:
        tm = Staged(trimap, float_only=False).dev.to(torch.int64).reshape(-1).contiguous()
    n_out = int((tm >= 0).sum().item())
    out = _ops.bilateral(1, M, N, params.sigma_length, params.sigma_angle, params.kernel_size,
                         params.iterations, fc_normals=_ops.stage_fc(nrm),
                         fc_centroids=_ops.centroids_f64(cen), trimap=tm, out_rows=n_out)[0]
    return S.give(out.to(x.dtype))


# north-star names (Polylidar3D / OrganizedPointFilters pybind API)
laplacian_opc = laplacian_filter_opc
bilateral_opc = bilateral_filter_opc
