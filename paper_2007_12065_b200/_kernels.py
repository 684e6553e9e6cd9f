"""Kernel boundary, mirroring flatpoly._kernels (reference: _kernels/__init__.py:9-30).

The reference picks a backend at import (Cython native | NumPy fallback).
Here there is exactly one backend: libopcfe on the GPU.  No fallback exists;
calls raise if the library or the device is missing.
"""

from __future__ import annotations

import torch

from . import _ops
from ._device import Staged

HAVE_NATIVE = True
ACTIVE = "cuda-sm100a"


def laplacian_filter(points, lam, kernel_size, iterations):
    """Same contract as _kernels.laplacian_filter (_native.pyx:225 / _fallback.py:82)."""
    from .smoothing import _laplacian_staged
    S = Staged(points)
    if S.dev.numel() == 0:                # the reference's loops run zero times: a copy
        return S.give(S.dev.clone())
    return _laplacian_staged(S, lam, kernel_size, iterations)


def bilateral_iterate(centroids, normals, sigma_length, sigma_angle, kernel_size, iterations):
    """Same contract as _kernels.bilateral_iterate (_native.pyx:287 / _fallback.py:120).

    Precision as smoothing.resolve_precision (float64 normals: the reference's fp64
    arithmetic by default)."""
    from .smoothing import BILATERAL_MAX_K32, resolve_precision
    C = Staged(centroids)
    Nn = Staged(normals)
    n = Nn.dev
    Mq, Nq = n.shape[:2]
    if n.numel() == 0:                    # the reference's loops run zero times: a copy
        return Nn.give(n.clone())
    if resolve_precision(None, n.dtype) == "strict" or kernel_size > BILATERAL_MAX_K32:
        out = _ops.bilateral_f64(C.dev.to(torch.float64), n.to(torch.float64), sigma_length,
                                 sigma_angle, kernel_size, iterations)
        return Nn.give(out.to(n.dtype))
    out = _ops.bilateral(1, Mq + 1, Nq + 1, sigma_length, sigma_angle, kernel_size, iterations,
                         fc_normals=_ops.stage_fc(n), fc_centroids=_ops.centroids_f64(C.dev))
    res = _ops.unstage_fc(out, 1, Mq, Nq, n.dtype, orig=n.unsqueeze(0).contiguous())[0]
    return Nn.give(res)


def find_cells(query_normals, ids_sorted, cell_normals, neighbors, slope, intercept,
               window_lo, window_hi):
    """Same contract as _kernels.find_cells (_native.pyx:120 / _fallback.py:14-44)."""
    from types import SimpleNamespace

    from .accumulator import DeviceAccumulator
    Q = Staged(query_normals)
    ga = SimpleNamespace(s2ids=ids_sorted, normals=cell_normals, neighbors=neighbors,
                         model_slope=slope, model_intercept=intercept, window_lo=window_lo,
                         window_hi=window_hi)
    return Q.give(DeviceAccumulator(ga).search(Q.dev.to(torch.float64)))


def grow_segment(triangles, halfedges, points, groups, visited, seed, label, anchor, normal,
                 ptp_max):
    """Same contract as _kernels.grow_segment (_native.pyx:170-222 / _fallback.py:47-80):
    the sorted members of the seed's segment; `visited` (uint8 [n_tri]) is updated in
    place -- a NumPy array on the host or a torch tensor on the device."""
    import numpy as np
    host = isinstance(visited, np.ndarray)
    dev = torch.device("cuda")
    G = Staged(groups, float_only=False).dev.to(torch.uint8)
    HE = Staged(halfedges, float_only=False).dev.to(torch.int64)
    check = float(ptp_max) > 0.0
    T = Staged(triangles, float_only=False).dev.to(torch.int64).reshape(-1, 3).contiguous() \
        if check else None
    P = Staged(points).dev.to(torch.float64).reshape(-1, 3).contiguous() if check else None
    V = torch.from_numpy(np.ascontiguousarray(visited)).to(dev) if host else visited
    m = _ops.grow_segment(T, HE, P, G, V, int(seed), int(label), np.asarray(anchor, np.float64),
                          np.asarray(normal, np.float64), float(ptp_max))
    if host:
        visited[...] = V.cpu().numpy()
        return m.cpu().numpy()
    return m
