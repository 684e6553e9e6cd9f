"""ctypes wrapper for oracle/opc_oracle.c -- TEST INFRASTRUCTURE ONLY.

Fast float64 restatement of the reference (see the C file header for the
file:line map).  Used by tests for parity at sizes where the NumPy oracle is
slow, and by bench.py as the multi-threaded CPU "port" baseline.  Pinned
against ``flatpoly_oracle`` and the golden vectors in tests/test_oracle.py.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libopc_oracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_lp = ctypes.POINTER(ctypes.c_int64)
_bp = ctypes.POINTER(ctypes.c_uint8)


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i, d = ctypes.c_int, ctypes.c_double
        L.oracle_laplacian.argtypes = [_dp, _dp, _dp, i, i, d, i, i]
        L.oracle_fc_data.argtypes = [_dp, i, i, _dp, _dp]
        L.oracle_bilateral.argtypes = [_dp, _dp, _dp, _dp, i, i, d, d, i, i]
        L.oracle_triangulate.argtypes = [_dp, i, i, _lp, _lp, _lp]
        L.oracle_triangulate.restype = ctypes.c_int64
        L.oracle_tri_normals.argtypes = [_dp, _lp, ctypes.c_int64, _dp]
        L.oracle_max_edge.argtypes = [_dp, _lp, ctypes.c_int64, d, _bp]
        L.oracle_group_assign.argtypes = [_dp, ctypes.c_int64, _dp, i, d, _bp, _bp]
        L.oracle_gather.argtypes = [_dp, _lp, ctypes.c_int64, _dp]
        _lib = L
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a, t):
    return a.ctypes.data_as(t)


def laplacian_filter(points, lam, kernel_size, iterations):
    src = _f64(points)
    M, N = src.shape[:2]
    out = np.empty_like(src)
    tmp = np.empty_like(src)
    lib().oracle_laplacian(_ptr(src, _dp), _ptr(out, _dp), _ptr(tmp, _dp), M, N,
                           float(lam), int(kernel_size), int(iterations))
    return out


def compute_fc_triangle_data(opc):
    src = _f64(opc)
    M, N = src.shape[:2]
    cen = np.empty((M - 1, N - 1, 2, 3))
    nrm = np.empty((M - 1, N - 1, 2, 3))
    lib().oracle_fc_data(_ptr(src, _dp), M, N, _ptr(cen, _dp), _ptr(nrm, _dp))
    return cen, nrm


def bilateral_iterate(centroids, normals, sigma_length, sigma_angle, kernel_size, iterations):
    c = _f64(centroids)
    n = _f64(normals)
    Mq, Nq = n.shape[:2]
    out = np.empty_like(n)
    tmp = np.empty_like(n)
    lib().oracle_bilateral(_ptr(c, _dp), _ptr(n, _dp), _ptr(out, _dp), _ptr(tmp, _dp),
                           Mq, Nq, float(sigma_length), float(sigma_angle),
                           int(kernel_size), int(iterations))
    return out


def triangulate(opc):
    """-> (triangles (T,3), trimap (G,), halfedges (3T,))"""
    src = _f64(opc)
    M, N = src.shape[:2]
    G = 2 * (M - 1) * (N - 1)
    trimap = np.empty(G, dtype=np.int64)
    tris = np.empty((G, 3), dtype=np.int64)
    he = np.empty(3 * G, dtype=np.int64)
    T = lib().oracle_triangulate(_ptr(src, _dp), M, N, _ptr(trimap, _lp), _ptr(tris, _lp),
                                 _ptr(he, _lp))
    return tris[:T].copy(), trimap, he[:3 * T].copy()


def triangle_normals(points, triangles):
    p = _f64(points).reshape(-1, 3)
    t = np.ascontiguousarray(triangles, dtype=np.int64)
    out = np.empty((len(t), 3))
    lib().oracle_tri_normals(_ptr(p, _dp), _ptr(t, _lp), len(t), _ptr(out, _dp))
    return out


def group_assignment(points, triangles, normals, dominant_normals, l_max, ang_min):
    """segmentation.py:52-74 (C restatement; BLAS FMA order for the scores)."""
    dn = np.ascontiguousarray(np.atleast_2d(dominant_normals), dtype=np.float64)
    if not 1 <= len(dn) <= 254:
        raise ValueError(f"need 1..254 dominant normals, got {len(dn)}")
    nrm = _f64(normals).reshape(-1, 3)
    flag = max_edge_mask(points, triangles, l_max).astype(np.uint8)
    out = np.empty(len(nrm), dtype=np.uint8)
    lib().oracle_group_assign(_ptr(nrm, _dp), len(nrm), _ptr(dn, _dp), len(dn), float(ang_min),
                              _ptr(flag, _bp), _ptr(out, _bp))
    return out


def max_edge_mask(points, triangles, l_max):
    p = _f64(points).reshape(-1, 3)
    t = np.ascontiguousarray(triangles, dtype=np.int64)
    out = np.empty(len(t), dtype=np.uint8)
    lib().oracle_max_edge(_ptr(p, _dp), _ptr(t, _lp), len(t), float(l_max), _ptr(out, _bp))
    return out.astype(bool)


def gather(fc_normals, trimap, n_tri):
    fc = _f64(fc_normals).reshape(-1, 3)
    tm = np.ascontiguousarray(trimap, dtype=np.int64)
    out = np.empty((n_tri, 3))
    lib().oracle_gather(_ptr(fc, _dp), _ptr(tm, _lp), len(tm), _ptr(out, _dp))
    return out


def front_end(opc, laplacian=None, bilateral=None, l_max=None):
    """pipeline.py:125-134 organized branch, C restatement."""
    opc = _f64(opc)
    if laplacian is not None:
        opc = laplacian_filter(opc, *laplacian)
    tris, trimap, he = triangulate(opc)
    pts = opc.reshape(-1, 3)
    out = dict(points=pts, triangles=tris, halfedges=he, trimap=trimap,
               grid_shape=opc.shape[:2], smoothed=opc)
    if bilateral is not None:
        cen, nrm = compute_fc_triangle_data(opc)
        sm = bilateral_iterate(cen, nrm, *bilateral)
        out["normals"] = gather(sm, trimap, len(tris))
    else:
        out["normals"] = triangle_normals(pts, tris)
    if l_max is not None:
        out["lmax_mask"] = max_edge_mask(pts, tris, l_max)
    return out


def s2_id(normals):
    """sfc.py:46-104 (C restatement, libm atan)."""
    q = _f64(normals).reshape(-1, 3)
    L = lib()
    L.oracle_s2id.restype = ctypes.c_uint64
    L.oracle_s2id.argtypes = [_dp]
    return np.array([L.oracle_s2id(_ptr(np.ascontiguousarray(r), _dp)) for r in q],
                    dtype=np.uint64)


def find_cells(query_normals, ids_sorted, cell_normals, neighbors, slope, intercept,
               window_lo, window_hi):
    """_kernels/_fallback.py:14-44 (C restatement)."""
    q = _f64(query_normals).reshape(-1, 3)
    ids = np.ascontiguousarray(ids_sorted, dtype=np.uint64)
    cn = _f64(cell_normals).reshape(-1, 3)
    nb = np.ascontiguousarray(neighbors, dtype=np.int64)
    out = np.empty(len(q), dtype=np.int64)
    L = lib()
    L.oracle_find_cells.argtypes = [_dp, ctypes.c_int64, ctypes.POINTER(ctypes.c_uint64), _dp,
                                    _lp, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_int64, ctypes.c_int64, _lp]
    L.oracle_find_cells(_ptr(q, _dp), len(q), ids.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                        _ptr(cn, _dp), _ptr(nb, _lp), len(ids), float(slope), float(intercept),
                        int(window_lo), int(window_hi), _ptr(out, _lp))
    return out


def integrate_normals(counts, normals, ids_sorted, cell_normals, neighbors, slope, intercept,
                      window_lo, window_hi, sample_pct=1.0):
    """accumulator.py:157-173: vote every round(1/sample_pct)-th finite normal."""
    normals = np.atleast_2d(np.asarray(normals, dtype=np.float64))
    stride = max(1, int(round(1.0 / sample_pct)))
    s = normals[::stride]
    s = s[np.all(np.isfinite(s), axis=1)]
    if len(s):
        idx = find_cells(s, ids_sorted, cell_normals, neighbors, slope, intercept,
                         window_lo, window_hi)
        counts = counts + np.bincount(idx, minlength=len(ids_sorted))
    return counts
