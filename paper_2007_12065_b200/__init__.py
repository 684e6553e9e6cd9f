"""paper_2007_12065_b200 -- B200-native organized-point-cloud front-end of Polylidar3D.

Drop-in for the hot path of the reference (flatpoly, arXiv 2007.12065):
implicit right-cut triangulation with GID map and twin half-edges, Laplacian
vertex smoothing, and bilateral filtering of triangle normals -- as hand-written
sm_100a CUDA kernels behind a C ABI (include/opcfe.h, lib/libopcfe.so).
There is no CPU fallback.
"""

from . import _kernels, accumulator, io, synthetic
from ._kernels import ACTIVE as kernel_backend
from .accumulator import (GaussianAccumulator, build_accumulator, find_cell_index,
                          find_cell_indices, integrate_normals)
from .frontend import FrontEnd, FrontEndResult, HostPipeline, front_end
from .geometry import DegenerateInputError, triangle_normals
from .mesh import (HalfEdgeMesh, compute_normals, extract_halfedges_opc, extract_triangles_opc,
                   extract_tri_mesh_from_organized_point_cloud, gid_of, gid_to_uvk, mesh_from_opc)
from .segmentation import (MAX_GROUPS, UNASSIGNED, SegmentationParams, extract_planar_segment,
                           group_assignment, grow_segments, max_edge_mask)
from .smoothing import (BilateralParams, LaplacianParams, bilateral_filter_opc, bilateral_opc,
                        compute_fc_triangle_data, get_precision, laplacian_filter_opc,
                        laplacian_opc, set_precision)
from .distributed import MultiDevicePipeline

__version__ = "0.1.0"

__all__ = [
    "kernel_backend", "FrontEnd", "FrontEndResult", "front_end", "DegenerateInputError",
    "triangle_normals", "HalfEdgeMesh", "compute_normals", "extract_halfedges_opc",
    "extract_triangles_opc", "extract_tri_mesh_from_organized_point_cloud", "gid_of",
    "gid_to_uvk", "mesh_from_opc", "UNASSIGNED", "MAX_GROUPS", "group_assignment",
    "max_edge_mask", "SegmentationParams", "extract_planar_segment", "grow_segments",
    "BilateralParams",
    "LaplacianParams", "bilateral_filter_opc", "bilateral_opc", "compute_fc_triangle_data",
    "laplacian_filter_opc", "laplacian_opc", "io", "set_precision", "get_precision",
    "MultiDevicePipeline", "GaussianAccumulator", "build_accumulator", "find_cell_index",
    "find_cell_indices", "integrate_normals",
]
