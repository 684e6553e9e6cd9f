"""libopcfe backend for flatpoly's kernel switch (flatpoly/_kernels/__init__.py:9-30).

A maintainer drops this file next to ``_native.pyx`` and applies
``integration/flatpoly_cuda.patch``; ``FLATPOLY_CUDA=1`` then selects it:

    FLATPOLY_CUDA=1 OPCFE_LIB=/path/to/libopcfe.so python -m pytest tests/

It binds the C ABI of ``include/opcfe.h`` with ctypes and the CUDA runtime only --
no torch, no new Python dependency.  Same functions, arguments, return values and
in-place effects as ``_native.pyx`` / ``_fallback.py``:

    laplacian_filter   (_native.pyx:225-284)  -> opcfe_laplacian_f64   (bit-exact)
    bilateral_iterate  (_native.pyx:287-364)  -> opcfe_bilateral_f64   (exp() last ulp)
    find_cells         (_native.pyx:120-167)  -> opcfe_find_cells
    grow_segment       (_native.pyx:170-222)  -> opcfe_grow_segment

plus the mesh / FC functions the patch routes here from mesh.py and smoothing.py
(plain NumPy in the reference, so they have no hook of their own):

    extract_triangles_opc   (mesh.py:58-96)       -> opcfe_stage_in + opcfe_triangulate
    extract_halfedges_opc   (mesh.py:99-135)      -> opcfe_halfedges_from_trimap
    triangle_normals        (geometry.py:134-147) -> opcfe_triangle_normals (bit-exact)
    compute_fc_triangle_data (smoothing.py:61-88) -> opcfe_fc_data (bit-exact)
    mesh_opc                (mesh.py:165-178)     -> one upload: triangles, trimap, twins and
                                                     normals of mesh_from_opc
    bilateral_filter_opc    (smoothing.py:91-114) -> FC data + filter + trimap gather on the
                                                     device (opcfe_bilateral_f64 scatter form)

Large results come back in pinned host blocks (a pool recycled as arrays are dropped):
a D2H into a fresh pageable NumPy array runs at ~2 GB/s, into pinned memory at the link
rate.  Device buffers come from a size-bucketed pool (no cudaFree per call).

Precision: the reference computes in float64, and so does this backend (the strict
kernels); ``FLATPOLY_CUDA=fast`` selects the fp32 Laplacian / bilateral kernels instead
(north-star 1e-5 contract, not bit-exact).
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref

import numpy as np

_vp, _i, _ll, _d, _f, _sz = (ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_double,
                             ctypes.c_float, ctypes.c_size_t)
_H2D, _D2H = 1, 2

FAST = os.environ.get("FLATPOLY_CUDA", "") == "fast"


def _load_cudart():
    for name in ("libcudart.so.12", "libcudart.so", "/usr/local/cuda/lib64/libcudart.so.12"):
        try:
            return ctypes.CDLL(name)
        except OSError:
            continue
    raise ImportError("FLATPOLY_CUDA: the CUDA runtime (libcudart.so.12) is not loadable")


_rt = _load_cudart()
_rt.cudaMalloc.argtypes = [ctypes.POINTER(_vp), _sz]
_rt.cudaFree.argtypes = [_vp]
_rt.cudaHostAlloc.argtypes = [ctypes.POINTER(_vp), _sz, ctypes.c_uint]
_rt.cudaFreeHost.argtypes = [_vp]
_rt.cudaMemcpy.argtypes = [_vp, _vp, _sz, _i]
_rt.cudaMemset.argtypes = [_vp, _i, _sz]
_rt.cudaDeviceSynchronize.argtypes = []
_rt.cudaGetErrorString.restype = ctypes.c_char_p

_op = ctypes.CDLL(os.environ.get("OPCFE_LIB", "libopcfe.so"))
_SIG = {
    "opcfe_last_error": (ctypes.c_char_p, []),
    "opcfe_points_pitch": (_i, [_i]),
    "opcfe_fc_pitch": (_i, [_i]),
    "opcfe_vmask_words": (_sz, [_i, _i, _i]),
    "opcfe_triangulate_workspace": (_sz, [_i, _i, _i]),
    "opcfe_stage_in": (_i, [_vp, _i, _ll, _ll, _i, _i, _i, _vp, _i, _vp, _vp]),
    "opcfe_unstage": (_i, [_vp, _i, _i, _i, _i, _vp, _i, _vp, _vp]),
    "opcfe_laplacian": (_i, [_vp, _vp, _vp, _vp, _i, _i, _i, _i, _f, _i, _i, _vp]),
    "opcfe_laplacian_f64": (_i, [_vp, _vp, _vp, _i, _i, _i, _d, _i, _i, _vp]),
    "opcfe_triangulate": (_i, [_vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _i, _vp, _d, _vp, _vp,
                               _sz, _vp]),
    "opcfe_halfedges_from_trimap": (_i, [_vp, _i, _i, ctypes.c_int64, _vp, _vp]),
    "opcfe_fc_data": (_i, [_vp, _i, _i, _i, _vp, _vp, _vp]),
    "opcfe_bilateral": (_i, [_vp, _i, _i, _i, _i, _vp, _vp, _f, _f, _i, _i, _vp, _vp, _vp, _vp,
                             _vp, _ll, _vp]),
    "opcfe_bilateral_f64": (_i, [_vp, _vp, _i, _i, _i, _d, _d, _i, _i, _vp, _vp, _vp, _vp, _vp,
                                 _ll, _vp]),
    "opcfe_triangle_normals": (_i, [_vp, _i, _vp, _ll, _vp, _vp]),
    "opcfe_trimap_stats": (_i, [_vp, _ll, _vp, _vp]),
    "opcfe_find_cells": (_i, [_vp, _ll, _ll, _vp, _vp, _vp, _ll, _d, _d, _ll, _ll, _vp, _vp,
                              _vp]),
    "opcfe_segments_workspace": (_sz, [_ll]),
    "opcfe_grow_segment": (_i, [_vp, _vp, _vp, _vp, _vp, _ll, _ll, _i, _vp, _vp, _d, _vp, _vp,
                                _vp, _sz, _vp]),
}
for _name, (_res, _args) in _SIG.items():
    _fn = getattr(_op, _name)
    _fn.restype, _fn.argtypes = _res, _args


def _check(rc, what):
    if rc != 0:
        msg = f"{what}: {_op.opcfe_last_error().decode(errors='replace')}"
        if rc == -1:
            raise ValueError(msg)
        if rc == -3:
            raise NotImplementedError(msg)
        raise RuntimeError(f"libopcfe error {rc}: {msg}")


class _Pool:
    """Size-bucketed (powers of two) cache of CUDA allocations: device buffers, or pinned
    host blocks.  Every call here ends with a synchronous copy on the legacy stream, so a
    released buffer is idle; cudaFree would synchronise the device on every call."""

    def __init__(self, name, alloc, free, cache_cap):
        self.name, self._alloc, self._free, self.cap = name, alloc, free, cache_cap
        self.free, self.cached, self.in_use = {}, 0, 0
        self.lock = threading.Lock()

    def get(self, nbytes):
        blk = 1 << max(int(nbytes) - 1, 15).bit_length()
        with self.lock:
            lst = self.free.get(blk)
            if lst:
                self.cached -= blk
                self.in_use += blk
                return lst.pop(), blk
        ptr = _vp()
        e = self._alloc(ctypes.byref(ptr), blk)
        if e != 0:
            raise MemoryError(f"{self.name}({blk}): {_rt.cudaGetErrorString(e).decode()}")
        with self.lock:
            self.in_use += blk
        return ptr, blk

    def put(self, ptr, blk):
        with self.lock:
            self.in_use -= blk
            if self.cached + blk <= self.cap:
                self.free.setdefault(blk, []).append(ptr)
                self.cached += blk
                return
        self._free(ptr)


_DEV = _Pool("cudaMalloc", _rt.cudaMalloc, _rt.cudaFree, 8 << 30)
_HOST = _Pool("cudaHostAlloc", lambda p, n: _rt.cudaHostAlloc(p, n, 0), _rt.cudaFreeHost, 4 << 30)
_PIN_MIN, _PIN_CAP = 4 << 20, int(os.environ.get("OPCFE_PINNED_OUT_MB", "4096")) << 20


def _host_empty(shape, dtype=np.float64):
    """A new host array for a large result: a view of a PINNED block (the D2H runs at the
    link rate instead of ~2 GB/s into fresh pageable memory), recycled once the array is
    garbage; plain np.empty below 4 MB or past OPCFE_PINNED_OUT_MB of results alive."""
    dtype = np.dtype(dtype)
    n = int(np.prod(shape))
    nbytes = n * dtype.itemsize
    if nbytes < _PIN_MIN or _HOST.in_use + 2 * nbytes > _PIN_CAP:
        return np.empty(shape, dtype)
    try:
        ptr, blk = _HOST.get(nbytes)
    except MemoryError:
        return np.empty(shape, dtype)
    raw = (ctypes.c_char * blk).from_address(ptr.value)
    arr = np.frombuffer(raw, dtype=dtype, count=n).reshape(shape)
    fin = weakref.finalize(raw, _HOST.put, ptr, blk)     # the array's base is `raw`
    fin.atexit = False
    return arr


class _Dev:
    """One device allocation (returned to the pool with the object)."""

    def __init__(self, nbytes):
        self.nbytes = max(int(nbytes), 16)
        self.ptr, self.blk = _DEV.get(self.nbytes)

    @classmethod
    def of(cls, arr):
        d = cls(arr.nbytes)
        if arr.nbytes:
            _sync_check(_rt.cudaMemcpy(d.ptr, arr.ctypes.data_as(_vp), arr.nbytes, _H2D))
        return d

    def get(self, arr):
        """Copy the first arr.nbytes back into `arr` (synchronous: the legacy stream)."""
        if arr.nbytes:
            _sync_check(_rt.cudaMemcpy(arr.ctypes.data_as(_vp), self.ptr, arr.nbytes, _D2H))
        return arr

    def __del__(self):
        if getattr(self, "ptr", None) is not None and self.ptr.value:
            try:
                _DEV.put(self.ptr, self.blk)
            except Exception:           # interpreter shutdown
                pass


def _sync_check(e):
    if e != 0:
        raise RuntimeError(f"CUDA: {_rt.cudaGetErrorString(e).decode()}")


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------- the _kernels functions
def laplacian_filter(points, lam, kernel_size, iterations):
    """_native.pyx:225-284 / _fallback.py:82-117."""
    src = _f64(points)
    if src.ndim != 3 or src.shape[2] != 3:
        raise ValueError("points must be an (M, N, 3) array")
    M, N = src.shape[:2]
    out = _host_empty(src.shape)
    if src.size == 0:
        return out
    d_in = _Dev.of(src)
    d_out = _Dev(src.nbytes)
    if FAST:
        pitch = _op.opcfe_points_pitch(N)
        grids = [_Dev(M * pitch * 4) for _ in range(3)]
        _check(_op.opcfe_stage_in(d_in.ptr, 1, 3 * N, 3 * M * N, 1, M, N, grids[0].ptr, pitch,
                                  None, None), "laplacian")
        _check(_op.opcfe_laplacian(grids[0].ptr, grids[1].ptr, grids[2].ptr, None, 1, M, N,
                                   pitch, float(lam), int(kernel_size), int(iterations), None),
               "laplacian")
        _check(_op.opcfe_unstage(grids[1].ptr, pitch, 1, M, N, d_out.ptr, 1, d_in.ptr, None),
               "laplacian")
    else:
        d_tmp = _Dev(src.nbytes) if iterations > 1 else None
        _check(_op.opcfe_laplacian_f64(d_in.ptr, d_out.ptr, d_tmp.ptr if d_tmp else None, 1, M,
                                       N, float(lam), int(kernel_size), int(iterations), None),
               "laplacian")
    return d_out.get(out)


def bilateral_iterate(centroids, normals, sigma_length, sigma_angle, kernel_size, iterations):
    """_native.pyx:287-364 / _fallback.py:120-166."""
    c, n = _f64(centroids), _f64(normals)
    Mq, Nq = n.shape[:2]
    out = _host_empty(n.shape)
    if n.size == 0:
        return out
    d_c, d_n, d_out = _Dev.of(c), _Dev.of(n), _Dev(n.nbytes)
    if FAST:
        fcp = _op.opcfe_fc_pitch(Nq + 1)
        fc = [_Dev(Mq * fcp * 4) for _ in range(4)]
        _check(_op.opcfe_stage_in(d_n.ptr, 1, 6 * Nq, 6 * Nq * Mq, 1, Mq, 2 * Nq, fc[0].ptr, fcp,
                                  None, None), "bilateral")
        _check(_op.opcfe_bilateral(None, 1, Mq + 1, Nq + 1, 0, fc[0].ptr, d_c.ptr,
                                   float(sigma_length), float(sigma_angle), int(kernel_size),
                                   int(iterations), fc[1].ptr, fc[2].ptr, fc[3].ptr, None, None,
                                   0, None), "bilateral")
        _check(_op.opcfe_unstage(fc[3].ptr, fcp, 1, Mq, 2 * Nq, d_out.ptr, 1, d_n.ptr, None),
               "bilateral")
    else:
        bufs = [_Dev(n.nbytes) if iterations > j else None for j in (1, 2)]
        _check(_op.opcfe_bilateral_f64(d_c.ptr, d_n.ptr, 1, Mq + 1, Nq + 1, float(sigma_length),
                                       float(sigma_angle), int(kernel_size), int(iterations),
                                       bufs[0].ptr if bufs[0] else None,
                                       bufs[1].ptr if bufs[1] else None, d_out.ptr, None, None,
                                       0, None), "bilateral")
    return d_out.get(out)


def find_cells(query_normals, ids_sorted, cell_normals, neighbors, slope, intercept,
               window_lo, window_hi):
    """_native.pyx:120-167 / _fallback.py:14-44: the accumulator cell of every query."""
    q = _f64(query_normals).reshape(-1, 3)
    ids = np.ascontiguousarray(ids_sorted, dtype=np.uint64)
    cn = _f64(cell_normals)
    nb = np.ascontiguousarray(neighbors, dtype=np.int64)
    out = np.empty(len(q), dtype=np.int64)
    if len(q) == 0:
        return out
    d_q, d_ids, d_cn, d_nb = _Dev.of(q), _Dev.of(ids), _Dev.of(cn), _Dev.of(nb)
    d_out = _Dev(out.nbytes)
    _check(_op.opcfe_find_cells(d_q.ptr, len(q), 1, d_ids.ptr, d_cn.ptr, d_nb.ptr, len(ids),
                                float(slope), float(intercept), int(window_lo), int(window_hi),
                                d_out.ptr, None, None), "find_cells")
    return d_out.get(out)


def grow_segment(triangles, halfedges, points, groups, visited, seed, label, anchor, normal,
                 ptp_max):
    """_native.pyx:170-222 / _fallback.py:47-80: sorted members of the seed's segment;
    `visited` (uint8) is updated in place."""
    he = np.ascontiguousarray(halfedges, dtype=np.int64)
    grp = np.ascontiguousarray(groups, dtype=np.uint8)
    n = len(grp)
    check = float(ptp_max) > 0.0
    d_t = _Dev.of(np.ascontiguousarray(triangles, dtype=np.int64)) if check else None
    d_p = _Dev.of(_f64(points)) if check else None
    d_he, d_g = _Dev.of(he), _Dev.of(grp)
    vis = np.ascontiguousarray(visited, dtype=np.uint8)
    d_v = _Dev.of(vis)
    ws_bytes = int(_op.opcfe_segments_workspace(n))
    d_ws = _Dev(ws_bytes)
    d_m, d_cnt = _Dev(8 * max(n, 1)), _Dev(8)
    a = (ctypes.c_double * 3)(*[float(x) for x in anchor])
    nn = (ctypes.c_double * 3)(*[float(x) for x in normal])
    _check(_op.opcfe_grow_segment(d_t.ptr if d_t else None, d_he.ptr, d_p.ptr if d_p else None,
                                  d_g.ptr, d_v.ptr, n, int(seed), int(label), a, nn,
                                  float(ptp_max), d_m.ptr, d_cnt.ptr, d_ws.ptr, ws_bytes, None),
           "grow_segment")
    cnt = d_cnt.get(np.empty(1, dtype=np.int64))[0]
    visited[...] = d_v.get(vis)
    return d_m.get(np.empty(int(cnt), dtype=np.int64))


# ---------------------------------------------------------------- mesh / FC functions
def extract_triangles_opc(opc):
    """mesh.py:58-96 (the caller has validated the shape): (triangles, trimap)."""
    src = _f64(opc)
    M, N = src.shape[:2]
    G = 2 * (M - 1) * (N - 1)
    d_src = _Dev.of(src)
    d_vm = _Dev(4 * _op.opcfe_vmask_words(1, M, N))
    _check(_op.opcfe_stage_in(d_src.ptr, 1, 3 * N, 3 * M * N, 1, M, N, None, 0, d_vm.ptr, None),
           "extract_triangles_opc")
    d_tm, d_tri, d_nt = _Dev(8 * G), _Dev(24 * G), _Dev(8)
    ws_bytes = int(_op.opcfe_triangulate_workspace(1, M, N))
    d_ws = _Dev(ws_bytes)
    _check(_op.opcfe_triangulate(d_vm.ptr, 1, M, N, d_tm.ptr, d_tri.ptr, None, d_nt.ptr, None, 0,
                                 None, -1.0, None, d_ws.ptr, ws_bytes, None),
           "extract_triangles_opc")
    T = int(d_nt.get(np.empty(1, dtype=np.int64))[0])
    return d_tri.get(_host_empty((T, 3), np.int64)), d_tm.get(_host_empty(G, np.int64))


def extract_halfedges_opc(trimap, M, N):
    """mesh.py:99-135 (the caller has validated the trimap's shape)."""
    tm = np.ascontiguousarray(trimap, dtype=np.int64).reshape(-1)
    if tm.size == 0:
        return np.full(0, -1, dtype=np.int64)
    d_tm, d_st = _Dev.of(tm), _Dev(16)
    _check(_op.opcfe_trimap_stats(d_tm.ptr, tm.size, d_st.ptr, None), "extract_halfedges_opc")
    n_tri = int(d_st.get(np.empty(2, dtype=np.int64))[1]) + 1        # trimap.max() + 1
    if n_tri <= 0:
        return np.full(0, -1, dtype=np.int64)
    he = _host_empty(3 * n_tri, np.int64)               # every entry written below
    d_he = _Dev(he.nbytes)
    _sync_check(_rt.cudaMemset(d_he.ptr, 0xFF, he.nbytes))          # -1 in every int64
    _check(_op.opcfe_halfedges_from_trimap(d_tm.ptr, int(M), int(N), n_tri, d_he.ptr, None),
           "extract_halfedges_opc")
    return d_he.get(he)


def triangle_normals(points, triangles):
    """geometry.py:134-147: unit normals, NaN for degenerate triangles (bit-exact)."""
    p = _f64(points).reshape(-1, 3)
    t = np.ascontiguousarray(triangles, dtype=np.int64).reshape(-1, 3)
    out = _host_empty((len(t), 3))
    if len(t) == 0:
        return out
    d_p, d_t, d_o = _Dev.of(p), _Dev.of(t), _Dev(out.nbytes)
    _check(_op.opcfe_triangle_normals(d_p.ptr, 1, d_t.ptr, len(t), d_o.ptr, None),
           "triangle_normals")
    return d_o.get(out)


def mesh_opc(opc):
    """mesh.py:165-178 in one upload (the caller has validated the shape): (triangles,
    trimap, halfedges, normals) -- extract_triangles_opc, extract_halfedges_opc and
    compute_normals of the reference, bit-identical."""
    src = _f64(opc)
    M, N = src.shape[:2]
    G = 2 * (M - 1) * (N - 1)
    d_src = _Dev.of(src)
    d_vm = _Dev(4 * _op.opcfe_vmask_words(1, M, N))
    _check(_op.opcfe_stage_in(d_src.ptr, 1, 3 * N, 3 * M * N, 1, M, N, None, 0, d_vm.ptr, None),
           "mesh_from_opc")
    d_tm, d_tri, d_he, d_nt = _Dev(8 * G), _Dev(24 * G), _Dev(24 * G), _Dev(8)
    ws_bytes = int(_op.opcfe_triangulate_workspace(1, M, N))
    d_ws = _Dev(ws_bytes)
    _check(_op.opcfe_triangulate(d_vm.ptr, 1, M, N, d_tm.ptr, d_tri.ptr, d_he.ptr, d_nt.ptr, None,
                                 0, None, -1.0, None, d_ws.ptr, ws_bytes, None), "mesh_from_opc")
    T = int(d_nt.get(np.empty(1, dtype=np.int64))[0])
    d_nrm = _Dev(24 * max(T, 1))
    if T:
        _check(_op.opcfe_triangle_normals(d_src.ptr, 1, d_tri.ptr, T, d_nrm.ptr, None),
               "mesh_from_opc")
    return (d_tri.get(_host_empty((T, 3), np.int64)), d_tm.get(_host_empty(G, np.int64)),
            d_he.get(_host_empty(3 * T, np.int64)), d_nrm.get(_host_empty((T, 3))))


def bilateral_filter_opc(opc, sigma_length, sigma_angle, kernel_size, iterations, trimap=None):
    """smoothing.py:91-114 (the caller has validated the shape and parameters): FC data,
    the bilateral iterations and the trimap gather on the device -- the fp64 kernels
    (strict); FLATPOLY_CUDA=fast keeps the reference's host gather over bilateral_iterate."""
    src = _f64(opc)
    M, N = src.shape[:2]
    if trimap is None:
        _, trimap = extract_triangles_opc(src)
    tm = np.ascontiguousarray(trimap, dtype=np.int64).reshape(-1)
    if FAST:
        cen, nrm = compute_fc_triangle_data(src)
        flat = bilateral_iterate(cen, nrm, sigma_length, sigma_angle, kernel_size,
                                 iterations).reshape(-1, 3)
        valid = tm >= 0
        out = np.empty((int(valid.sum()), 3))
        out[tm[valid]] = flat[valid]
        return out
    d_tm, d_st = _Dev.of(tm), _Dev(16)
    _check(_op.opcfe_trimap_stats(d_tm.ptr, tm.size, d_st.ptr, None), "bilateral_filter_opc")
    T, top = (int(x) for x in d_st.get(np.empty(2, dtype=np.int64)))   # valid.sum(), max
    if top >= T:                            # out[trimap[valid]] out of bounds (numpy's error)
        raise IndexError(f"index {top} is out of bounds for axis 0 with size {T}")
    out = _host_empty((T, 3))
    if T == 0:
        return out
    Mq, Nq = M - 1, N - 1
    fc = Mq * Nq * 6 * 8
    d_src = _Dev.of(src)
    d_c, d_n, d_out = _Dev(fc), _Dev(fc), _Dev(out.nbytes)
    _check(_op.opcfe_fc_data(d_src.ptr, 1, M, N, d_c.ptr, d_n.ptr, None), "bilateral_filter_opc")
    bufs = [_Dev(fc) if iterations > j else None for j in (1, 2)]
    _check(_op.opcfe_bilateral_f64(d_c.ptr, d_n.ptr, 1, M, N, float(sigma_length),
                                   float(sigma_angle), int(kernel_size), int(iterations),
                                   bufs[0].ptr if bufs[0] else None,
                                   bufs[1].ptr if bufs[1] else None, None, d_tm.ptr, d_out.ptr,
                                   T, None), "bilateral_filter_opc")
    return d_out.get(out)


def compute_fc_triangle_data(opc):
    """smoothing.py:61-88 (the caller has validated the shape): (centroids, normals)."""
    src = _f64(opc)
    M, N = src.shape[:2]
    cen = _host_empty((M - 1, N - 1, 2, 3))
    nrm = _host_empty((M - 1, N - 1, 2, 3))
    d_src, d_c, d_n = _Dev.of(src), _Dev(cen.nbytes), _Dev(nrm.nbytes)
    _check(_op.opcfe_fc_data(d_src.ptr, 1, M, N, d_c.ptr, d_n.ptr, None),
           "compute_fc_triangle_data")
    return d_c.get(cen), d_n.get(nrm)
