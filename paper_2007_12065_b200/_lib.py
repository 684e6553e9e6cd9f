"""ctypes binding of libopcfe.so (the C ABI declared in include/opcfe.h).

This is the product's only compute path.  There is no CPU fallback: if the
library is missing or no CUDA device is present, every compute call raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# OPCFE_LIB: an alternative in-tree build of the same library (kernel A/B experiments)
LIB_PATH = os.environ.get("OPCFE_LIB") or os.path.join(PKG_DIR, "lib", "libopcfe.so")

OPCFE_OK = 0
OPCFE_ERR_INVALID = -1
OPCFE_ERR_CUDA = -2
OPCFE_ERR_UNSUPPORTED = -3
OPCFE_ERR_WORKSPACE = -4
OPCFE_ERR_DRIVER = -5

# every symbol include/opcfe.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "opcfe_version", "opcfe_last_error", "opcfe_points_pitch", "opcfe_fc_pitch",
    "opcfe_vmask_words", "opcfe_triangulate_workspace", "opcfe_stage_in", "opcfe_unstage",
    "opcfe_laplacian",
    "opcfe_triangulate", "opcfe_halfedges_from_trimap", "opcfe_fc_data", "opcfe_bilateral",
    "opcfe_triangle_normals", "opcfe_find_cells", "opcfe_group_assignment", "opcfe_max_edge_mask", "opcfe_front_end_workspace",
    "opcfe_front_end", "opcfe_front_end_profiled", "opcfe_segments_workspace",
    "opcfe_grow_segment", "opcfe_segment_components",
    "opcfe_laplacian_f64", "opcfe_fc_data_f64", "opcfe_bilateral_f64", "opcfe_narrow_indices",
    "opcfe_trimap_stats", "opcfe_laplacian_mixed",
)

PRECISION_FAST = 0      # OPCFE_PRECISION_FAST
PRECISION_STRICT = 1    # OPCFE_PRECISION_STRICT
PRECISION_MIXED = 2     # OPCFE_PRECISION_MIXED


class FrontEndParams(ctypes.Structure):
    """opcfe_front_end_params (include/opcfe.h)."""
    _fields_ = [
        ("laplacian_iterations", ctypes.c_int),
        ("laplacian_kernel_size", ctypes.c_int),
        ("laplacian_lambda", ctypes.c_double),
        ("bilateral_iterations", ctypes.c_int),
        ("bilateral_kernel_size", ctypes.c_int),
        ("sigma_length", ctypes.c_double),
        ("sigma_angle", ctypes.c_double),
        ("l_max", ctypes.c_double),
        ("dominant_normals", ctypes.c_void_p),
        ("n_dominant", ctypes.c_int),
        ("ang_min", ctypes.c_double),
        ("precision", ctypes.c_int),
    ]


class FrontEndIO(ctypes.Structure):
    """opcfe_front_end_io (include/opcfe.h)."""
    _fields_ = [
        ("src", ctypes.c_void_p),
        ("src_kind", ctypes.c_int),
        ("src_pitch", ctypes.c_int),
        ("points", ctypes.c_void_p),
        ("trimap", ctypes.c_void_p),
        ("triangles", ctypes.c_void_p),
        ("halfedges", ctypes.c_void_p),
        ("normals", ctypes.c_void_p),
        ("lmax_flag", ctypes.c_void_p),
        ("n_tri", ctypes.c_void_p),
        ("labels", ctypes.c_void_p),
    ]


_lib = None
_lock = threading.Lock()


class OpcfeError(RuntimeError):
    """A libopcfe call failed (CUDA error, unsupported configuration, ...)."""


def build(jobs: int = 8) -> str:
    """Compile libopcfe.so for sm_100a (nvcc cross-compiles without a GPU)."""
    subprocess.run(["make", "-s", "-C", PKG_DIR, f"-j{jobs}"], check=True)
    return LIB_PATH


def _declare(L):
    vp, i, ll, d, f = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_double, ctypes.c_float
    sz = ctypes.c_size_t
    sig = {
        "opcfe_version": (i, []),
        "opcfe_last_error": (ctypes.c_char_p, []),
        "opcfe_points_pitch": (i, [i]),
        "opcfe_fc_pitch": (i, [i]),
        "opcfe_vmask_words": (sz, [i, i, i]),
        "opcfe_triangulate_workspace": (sz, [i, i, i]),
        "opcfe_stage_in": (i, [vp, i, ll, ll, i, i, i, vp, i, vp, vp]),
        "opcfe_unstage": (i, [vp, i, i, i, i, vp, i, vp, vp]),
        "opcfe_laplacian": (i, [vp, vp, vp, vp, i, i, i, i, f, i, i, vp]),
        "opcfe_triangulate": (i, [vp, i, i, i, vp, vp, vp, vp, vp, i, vp, d, vp, vp, sz, vp]),
        "opcfe_halfedges_from_trimap": (i, [vp, i, i, ctypes.c_int64, vp, vp]),
        "opcfe_fc_data": (i, [vp, i, i, i, vp, vp, vp]),
        "opcfe_bilateral": (i, [vp, i, i, i, i, vp, vp, f, f, i, i, vp, vp, vp, vp, vp, ll, vp]),
        "opcfe_triangle_normals": (i, [vp, i, vp, ll, vp, vp]),
        "opcfe_max_edge_mask": (i, [vp, i, vp, ll, d, vp, vp]),
        "opcfe_find_cells": (i, [vp, ll, ll, vp, vp, vp, ll, d, d, ll, ll, vp, vp, vp]),
        "opcfe_group_assignment": (i, [vp, i, ll, i, vp, vp, i, d, vp, vp, vp]),
        "opcfe_segments_workspace": (sz, [ll]),
        "opcfe_grow_segment": (i, [vp, vp, vp, vp, vp, ll, ll, i, vp, vp, d, vp, vp, vp, sz, vp]),
        "opcfe_segment_components": (i, [vp, vp, ll, vp, vp, vp, sz, vp]),
        "opcfe_narrow_indices": (i, [vp, vp, i, ll, i, vp, ll, ll, vp]),
        "opcfe_trimap_stats": (i, [vp, ll, vp, vp]),
        "opcfe_laplacian_f64": (i, [vp, vp, vp, i, i, i, d, i, i, vp]),
        "opcfe_laplacian_mixed": (i, [vp, vp, vp, i, i, i, d, i, i, vp]),
        "opcfe_fc_data_f64": (i, [vp, i, i, i, vp, vp, vp]),
        "opcfe_bilateral_f64": (i, [vp, vp, i, i, i, d, d, i, i, vp, vp, vp, vp, vp, ll, vp]),
        "opcfe_front_end_workspace": (sz, [i, i, i, ctypes.POINTER(FrontEndParams), i, i]),
        "opcfe_front_end": (i, [i, i, i, ctypes.POINTER(FrontEndParams),
                                ctypes.POINTER(FrontEndIO), vp, sz, vp]),
        "opcfe_front_end_profiled": (i, [i, i, i, ctypes.POINTER(FrontEndParams),
                                         ctypes.POINTER(FrontEndIO), vp, sz, vp,
                                         ctypes.POINTER(ctypes.c_void_p)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args


def lib():
    """Load libopcfe.so (building it first if this checkout has no binary)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    build()
                L = ctypes.CDLL(LIB_PATH)
                _declare(L)
                _lib = L
    return _lib


def check(rc: int, what: str = "opcfe") -> None:
    if rc != OPCFE_OK:
        msg = lib().opcfe_last_error().decode(errors="replace")
        if rc == OPCFE_ERR_INVALID:
            raise ValueError(f"{what}: {msg}")
        if rc == OPCFE_ERR_UNSUPPORTED:
            raise NotImplementedError(f"{what}: {msg}")
        raise OpcfeError(f"{what} failed ({rc}): {msg}")
