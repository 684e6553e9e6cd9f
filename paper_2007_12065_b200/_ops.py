"""Device-level operations: torch CUDA tensors in, torch CUDA tensors out.

Thin wrappers over the libopcfe C ABI (include/opcfe.h).  Every function
enqueues work on torch's current stream and never synchronises, except where
a data-dependent output size must be read back (n_tri), which is explicit.
Grids are (F, M, N, 3) or (M, N, 3); internally fp32 rows padded to
``points_pitch(N)`` floats (the TMA row-stride rule).
"""

from __future__ import annotations

import torch

from . import _lib
from ._device import fc_pitch, points_pitch, ptr, stream


def _frames(x: torch.Tensor):
    if x.dim() == 3:
        return 1, x.shape[0], x.shape[1]
    return x.shape[0], x.shape[1], x.shape[2]


def stage_in(src: torch.Tensor, want_points=True, want_mask=True):
    """(F,M,N,3)|(M,N,3) f32/f64 contiguous -> (padded fp32 grid [F,M,pitch], vmask)."""
    F, M, N = _frames(src)
    L = _lib.lib()
    pitch = points_pitch(N)
    dst = torch.empty((F, M, pitch), dtype=torch.float32, device=src.device) if want_points else None
    vmask = torch.empty(int(L.opcfe_vmask_words(F, M, N)), dtype=torch.int32,
                        device=src.device) if want_mask else None
    _lib.check(L.opcfe_stage_in(src.data_ptr(), int(src.dtype == torch.float64), 3 * N,
                                3 * N * M, F, M, N, ptr(dst), pitch, ptr(vmask), stream()),
               "stage_in")
    return dst, vmask


def unstage(grid: torch.Tensor, F: int, M: int, N: int, dtype, orig: torch.Tensor | None = None):
    """padded fp32 grid -> contiguous (F,M,N,3) of `dtype`; unchanged values restored from orig."""
    out = torch.empty((F, M, N, 3), dtype=dtype, device=grid.device)
    if orig is not None:
        assert orig.dtype == dtype and orig.is_contiguous()
    _lib.check(_lib.lib().opcfe_unstage(grid.data_ptr(), grid.shape[-1], F, M, N, out.data_ptr(),
                                        int(dtype == torch.float64), ptr(orig), stream()),
               "unstage")
    return out


def laplacian(grid: torch.Tensor, F: int, M: int, N: int, lam: float, kernel_size: int,
              iterations: int, vmask: torch.Tensor | None = None, out: torch.Tensor | None = None):
    """Iterated Laplacian on a padded fp32 grid; returns the padded result."""
    out = torch.empty_like(grid) if out is None else out
    tmp = torch.empty_like(grid) if iterations > 1 else None
    _lib.check(_lib.lib().opcfe_laplacian(grid.data_ptr(), out.data_ptr(), ptr(tmp), ptr(vmask),
                                          F, M, N, grid.shape[-1], float(lam), int(kernel_size),
                                          int(iterations), stream()),
               "laplacian")
    return out


def triangulate(vmask: torch.Tensor, F: int, M: int, N: int, halfedges=True, grid=None,
                normals=False, l_max=None):
    """One-pass triangulation.  Returns dict of capacity-sized device arrays + n_tri (device)."""
    dev = vmask.device
    G = 2 * (M - 1) * (N - 1)
    L = _lib.lib()
    out = {
        "trimap": torch.empty((F, G), dtype=torch.int64, device=dev),
        "triangles": torch.empty((F, G, 3), dtype=torch.int64, device=dev),
        "halfedges": torch.empty((F, G * 3), dtype=torch.int64, device=dev) if halfedges else None,
        "n_tri": torch.empty((F,), dtype=torch.int64, device=dev),
        "normals": torch.empty((F, G, 3), dtype=torch.float32, device=dev) if normals else None,
        "lmax_flag": torch.empty((F, G), dtype=torch.uint8, device=dev) if l_max is not None else None,
    }
    ws_bytes = int(L.opcfe_triangulate_workspace(F, M, N))
    ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device=dev)
    pitch = grid.shape[-1] if grid is not None else 0
    _lib.check(L.opcfe_triangulate(vmask.data_ptr(), F, M, N, out["trimap"].data_ptr(),
                                   out["triangles"].data_ptr(), ptr(out["halfedges"]),
                                   out["n_tri"].data_ptr(), ptr(grid), pitch, ptr(out["normals"]),
                                   float(l_max) if l_max is not None else -1.0,
                                   ptr(out["lmax_flag"]), ws.data_ptr(), ws_bytes, stream()),
               "triangulate")
    return out


def halfedges_from_trimap(trimap: torch.Tensor, M: int, N: int, n_tri: int):
    he = torch.full((3 * max(n_tri, 0),), -1, dtype=torch.int64, device=trimap.device)
    if n_tri > 0:
        _lib.check(_lib.lib().opcfe_halfedges_from_trimap(trimap.data_ptr(), M, N, n_tri,
                                                          he.data_ptr(), stream()),
                   "halfedges_from_trimap")
    return he


def trimap_stats(trimap: torch.Tensor):
    """(valid-entry count, largest entry) of an int64 GID map (opcfe_trimap_stats)."""
    st = torch.empty(2, dtype=torch.int64, device=trimap.device)
    _lib.check(_lib.lib().opcfe_trimap_stats(trimap.data_ptr(), trimap.numel(), st.data_ptr(),
                                             stream()), "trimap_stats")
    cnt, mx = st.tolist()
    return cnt, mx


def fc_data(opc: torch.Tensor):
    """(M,N,3) f32/f64 contiguous -> centroids, normals (M-1,N-1,2,3) same dtype."""
    M, N = opc.shape[:2]
    cen = torch.empty((M - 1, N - 1, 2, 3), dtype=opc.dtype, device=opc.device)
    nrm = torch.empty_like(cen)
    _lib.check(_lib.lib().opcfe_fc_data(opc.data_ptr(), int(opc.dtype == torch.float64), M, N,
                                        cen.data_ptr(), nrm.data_ptr(), stream()),
               "fc_data")
    return cen, nrm


def bilateral(F: int, M: int, N: int, sigma_length: float, sigma_angle: float, kernel_size: int,
              iterations: int, grid=None, fc_normals=None, fc_centroids=None, trimap=None,
              out_rows=None):
    """Bilateral normal filter.

    Input either the padded point grid (normals fused into iteration 1) or padded
    FC arrays [F, M-1, fc_pitch].  With ``trimap`` the last iteration scatters into
    mesh order ([F, out_rows, 3]); otherwise returns padded FC normals.
    """
    dev = (grid if grid is not None else fc_normals).device
    fcp = fc_pitch(N)
    shape_fc = (F, M - 1, fcp)
    buf_a = torch.empty(shape_fc, dtype=torch.float32, device=dev) if iterations > 1 else None
    buf_b = torch.empty(shape_fc, dtype=torch.float32, device=dev) if iterations > 2 else None
    out_fc = out_mesh = None
    if trimap is not None:
        out_mesh = torch.empty((F, out_rows, 3), dtype=torch.float32, device=dev)
    else:
        out_fc = torch.empty(shape_fc, dtype=torch.float32, device=dev)
    pitch = grid.shape[-1] if grid is not None else 0
    _lib.check(_lib.lib().opcfe_bilateral(ptr(grid), F, M, N, pitch, ptr(fc_normals),
                                          ptr(fc_centroids), float(sigma_length),
                                          float(sigma_angle), int(kernel_size), int(iterations),
                                          ptr(buf_a), ptr(buf_b), ptr(out_fc), ptr(trimap),
                                          ptr(out_mesh), int(out_rows or 0), stream()),
               "bilateral")
    return out_mesh if trimap is not None else out_fc


def stage_fc(arr: torch.Tensor):
    """(F?,Mq,Nq,2,3) contiguous -> padded fp32 FC rows [F, Mq, fc_pitch]."""
    if arr.dim() == 4:
        arr = arr.unsqueeze(0)
    F, Mq, Nq = arr.shape[:3]
    # an FC row of Nq quads is 2*Nq xyz triplets: reuse the grid stager
    grid, _ = stage_in(arr.reshape(F, Mq, 2 * Nq, 3), want_points=True, want_mask=False)
    return grid


def centroids_f64(arr: torch.Tensor):
    """(F?,Mq,Nq,2,3) -> contiguous float64 [F, Mq, Nq, 2, 3] (opcfe_bilateral's centroids)."""
    if arr.dim() == 4:
        arr = arr.unsqueeze(0)
    return arr.to(torch.float64).contiguous()


def unstage_fc(fc: torch.Tensor, F: int, Mq: int, Nq: int, dtype, orig=None):
    out = unstage(fc, F, Mq, 2 * Nq, dtype,
                  None if orig is None else orig.reshape(F, Mq, 2 * Nq, 3))
    return out.reshape(F, Mq, Nq, 2, 3)


def triangle_normals(points: torch.Tensor, triangles: torch.Tensor):
    T = triangles.shape[0]
    out = torch.empty((T, 3), dtype=points.dtype, device=points.device)
    _lib.check(_lib.lib().opcfe_triangle_normals(points.data_ptr(),
                                                 int(points.dtype == torch.float64),
                                                 triangles.data_ptr(), T, out.data_ptr(), stream()),
               "triangle_normals")
    return out


def group_assignment(normals: torch.Tensor, dominant: torch.Tensor, ang_min: float,
                     lflag: torch.Tensor | None = None, n_tri: torch.Tensor | None = None):
    """(F?, T, 3) normals (f32/f64) x (G, 3) f64 dominant normals -> uint8 labels (F?, T)."""
    batched = normals.dim() == 3
    F = normals.shape[0] if batched else 1
    T = normals.shape[-2]
    out = torch.empty(normals.shape[:-1], dtype=torch.uint8, device=normals.device)
    dn = dominant.to(device=normals.device, dtype=torch.float64).contiguous()
    _lib.check(_lib.lib().opcfe_group_assignment(normals.data_ptr(),
                                                 int(normals.dtype == torch.float64), T, F,
                                                 ptr(n_tri), dn.data_ptr(), dn.shape[0],
                                                 float(ang_min), ptr(lflag), out.data_ptr(),
                                                 stream()),
               "group_assignment")
    return out


def max_edge_mask(points: torch.Tensor, triangles: torch.Tensor, l_max: float):
    T = triangles.shape[0]
    out = torch.empty((T,), dtype=torch.uint8, device=points.device)
    _lib.check(_lib.lib().opcfe_max_edge_mask(points.data_ptr(), int(points.dtype == torch.float64),
                                              triangles.data_ptr(), T, float(l_max),
                                              out.data_ptr(), stream()),
               "max_edge_mask")
    return out.bool()


# ------------------------------------------------------------------ region growing
def _seg_ws(n_tri: int, device) -> torch.Tensor:
    nb = int(_lib.lib().opcfe_segments_workspace(n_tri))
    return torch.empty((max(nb, 1),), dtype=torch.uint8, device=device)


def grow_segment(triangles, halfedges, points, groups, visited, seed: int, label: int,
                 anchor, normal, ptp_max: float):
    """Device tensors in; sorted int64 members (device) out; `visited` updated in place."""
    import ctypes
    n = int(groups.shape[0])
    ws = _seg_ws(n, groups.device)
    members = torch.empty((n,), dtype=torch.int64, device=groups.device)
    cnt = torch.empty((1,), dtype=torch.int64, device=groups.device)
    a = (ctypes.c_double * 3)(*[float(x) for x in anchor])
    nn = (ctypes.c_double * 3)(*[float(x) for x in normal])
    _lib.check(_lib.lib().opcfe_grow_segment(ptr(triangles), halfedges.data_ptr(), ptr(points),
                                             groups.data_ptr(), visited.data_ptr(), n, int(seed),
                                             int(label), a, nn, float(ptp_max),
                                             members.data_ptr(), cnt.data_ptr(), ws.data_ptr(),
                                             ws.numel(), stream()),
               "grow_segment")
    return members[: int(cnt.item())]


def segment_components(halfedges, groups, with_size: bool = True):
    """(component root = min index or -1, size at the root) per triangle (device)."""
    n = int(groups.shape[0])
    ws = _seg_ws(n, groups.device)
    comp = torch.empty((n,), dtype=torch.int64, device=groups.device)
    size = torch.empty((n,), dtype=torch.int64, device=groups.device) if with_size else None
    _lib.check(_lib.lib().opcfe_segment_components(halfedges.data_ptr(), groups.data_ptr(), n,
                                                   comp.data_ptr(), ptr(size), ws.data_ptr(),
                                                   ws.numel(), stream()),
               "segment_components")
    return comp, size


# ------------------------------------------------------------------ strict (fp64) kernels
def laplacian_f64(x: torch.Tensor, lam: float, kernel_size: int, iterations: int,
                  out: torch.Tensor | None = None, mixed: bool = False):
    """(F?, M, N, 3) float64 contiguous -> smoothed grid (same shape), the reference's own
    fp64 arithmetic (opcfe_laplacian_f64: bit-exact), any odd kernel size; mixed: rsqrt pair
    weights (opcfe_laplacian_mixed: a few ulp)."""
    x = x.contiguous()
    F, M, N = _frames(x)
    out = torch.empty_like(x) if out is None else out
    tmp = torch.empty_like(x) if iterations > 1 else None
    fn = _lib.lib().opcfe_laplacian_mixed if mixed else _lib.lib().opcfe_laplacian_f64
    _lib.check(fn(x.data_ptr(), out.data_ptr(), ptr(tmp), F, M, N, float(lam), int(kernel_size),
                  int(iterations), stream()),
               "laplacian")
    return out


def fc_data_f64(x: torch.Tensor):
    """(F?, M, N, 3) float64 -> centroids, normals (F?, M-1, N-1, 2, 3) float64 (bit-exact)."""
    x = x.contiguous()
    F, M, N = _frames(x)
    shape = (M - 1, N - 1, 2, 3) if x.dim() == 3 else (F, M - 1, N - 1, 2, 3)
    cen = torch.empty(shape, dtype=torch.float64, device=x.device)
    nrm = torch.empty_like(cen)
    _lib.check(_lib.lib().opcfe_fc_data_f64(x.data_ptr(), F, M, N, cen.data_ptr(), nrm.data_ptr(),
                                            stream()),
               "fc_data")
    return cen, nrm


def bilateral_f64(centroids: torch.Tensor, normals: torch.Tensor, sigma_length: float,
                  sigma_angle: float, kernel_size: int, iterations: int, trimap=None,
                  out_rows=None):
    """FC arrays (F?, Mq, Nq, 2, 3) float64 -> filtered FC normals (same shape), or with
    ``trimap`` ((F?, G) int64) the mesh-order normals (F?, out_rows, 3)
    (opcfe_bilateral_f64: the reference's fp64 arithmetic, any odd kernel size)."""
    batched = normals.dim() == 5
    c = centroids.contiguous() if batched else centroids.contiguous().unsqueeze(0)
    n = normals.contiguous() if batched else normals.contiguous().unsqueeze(0)
    F, Mq, Nq = n.shape[:3]
    buf_a = torch.empty_like(n) if iterations > 1 else None
    buf_b = torch.empty_like(n) if iterations > 2 else None
    out_fc = out_mesh = None
    if trimap is not None:
        out_mesh = torch.empty((F, int(out_rows), 3), dtype=torch.float64, device=n.device)
        tm = trimap.reshape(F, -1).contiguous()
        if tm.shape[1] != 2 * Mq * Nq:
            from .geometry import DegenerateInputError
            raise DegenerateInputError("trimap does not match the grid shape")
    else:
        out_fc = torch.empty_like(n)
        tm = None
    _lib.check(_lib.lib().opcfe_bilateral_f64(c.data_ptr(), n.data_ptr(), F, Mq + 1, Nq + 1,
                                              float(sigma_length), float(sigma_angle),
                                              int(kernel_size), int(iterations), ptr(buf_a),
                                              ptr(buf_b), ptr(out_fc), ptr(tm), ptr(out_mesh),
                                              int(out_rows or 0), stream()),
               "bilateral")
    res = out_mesh if trimap is not None else out_fc
    return res if batched else res[0]
