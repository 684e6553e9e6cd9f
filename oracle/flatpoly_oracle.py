"""CPU oracle for the organized-point-cloud (OPC) front-end -- TEST INFRASTRUCTURE ONLY.

This module is a NumPy restatement of the reference's (flatpoly) algorithms for
the hot path.  It is the *checker*: only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product package (``paper_2007_12065_b200``) never imports it and has no CPU
fallback.

Every function cites the reference file:line it restates (paths relative to
``/root/reference/pkg/src/flatpoly``).  All arithmetic is float64 and follows
the reference's operation order so that integer outputs are bit-exact and
float outputs agree to the last ulp (except ``exp`` in the bilateral filter).

Pinning: ``tests/test_oracle.py`` checks every function here against the golden
vectors in ``tests/golden/*.npz``; those were produced by importing the real
reference (NumPy backend = semantics of record, ``_kernels/_fallback.py:3-4``,
plus its compiled Cython backend) with ``tests/golden/make_golden.py``.
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "laplacian_filter", "bilateral_iterate", "extract_triangles_opc",
    "extract_halfedges_opc", "triangle_normals", "compute_fc_triangle_data",
    "bilateral_filter_opc", "mesh_from_opc", "max_edge_mask", "front_end",
    "gid_of", "gid_to_uvk",
]


# --------------------------------------------------------------------------- ids
def gid_of(u, v, k, N):
    """GID of FC triangle (u, v, k): mesh.py:46-48."""
    return 2 * (u * (N - 1) + v) + k


def gid_to_uvk(gid, N):
    """Inverse of gid_of: mesh.py:51-55."""
    q, k = divmod(gid, 2)
    u, v = divmod(q, N - 1)
    return u, v, k


# -------------------------------------------------------------------- Laplacian
def laplacian_filter(points, lam, kernel_size, iterations):
    """Inverse-distance Laplacian on the (M, N, 3) grid.

    Restates ``_kernels/_fallback.py:82-117`` (== ``_native.pyx:225-284``):
    per interior vertex, neighbours in the (2h+1)^2 window (du outer, dv
    inner, self excluded, off-grid skipped) with finite non-zero distance get
    weight 1/dist; update p + (lam/wsum)*sum(w*d).  NaN/inf centres, vertices
    with wsum == 0 and the outer 1-px ring are copied unchanged.
    """
    cur = np.array(points, dtype=np.float64, copy=True)
    M, N = cur.shape[:2]
    h = kernel_size // 2
    for _ in range(iterations):
        acc = np.zeros_like(cur)
        wsum = np.zeros((M, N))
        for du in range(-h, h + 1):
            for dv in range(-h, h + 1):
                if du == 0 and dv == 0:
                    continue
                # destination window [u_lo, u_hi) x [v_lo, v_hi) whose
                # neighbour (u+du, v+dv) is on the grid
                u_lo, u_hi = max(0, -du), min(M, M - du)
                v_lo, v_hi = max(0, -dv), min(N, N - dv)
                if u_lo >= u_hi or v_lo >= v_hi:
                    continue
                ctr = cur[u_lo:u_hi, v_lo:v_hi]
                nbr = cur[u_lo + du:u_hi + du, v_lo + dv:v_hi + dv]
                d = nbr - ctr
                dist = np.sqrt(d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]
                               + d[..., 2] * d[..., 2])
                use = np.isfinite(dist) & (dist > 0.0)
                w = np.zeros_like(dist)
                w[use] = 1.0 / dist[use]
                a = acc[u_lo:u_hi, v_lo:v_hi]
                a[use] += d[use] * w[use][:, None]
                wsum[u_lo:u_hi, v_lo:v_hi] += w
        nxt = cur.copy()
        move = (wsum > 0.0) & np.isfinite(cur).all(axis=2)
        move[0, :] = move[-1, :] = False
        move[:, 0] = move[:, -1] = False
        nxt[move] = cur[move] + (lam / wsum[move])[:, None] * acc[move]
        cur = nxt
    return cur


# ----------------------------------------------------------------- triangulation
def _quad_validity(opc):
    """Per-quad (first, second) validity: mesh.py:69,78-82 (NaN/inf => invalid)."""
    ok = np.isfinite(opc).all(axis=2)
    p1, p2 = ok[:-1, :-1], ok[:-1, 1:]
    p3, p4 = ok[1:, 1:], ok[1:, :-1]
    return p1 & p2 & p3, p1 & p3 & p4


def extract_triangles_opc(opc):
    """Right-cut triangles in GID order + GID->triangle map: mesh.py:58-96.

    first = {p3, p2, p1} iff p1, p2, p3 finite; second = {p1, p4, p3} iff
    p1, p3, p4 finite; trimap[gid] = running count of valid GIDs before gid.
    """
    opc = np.asarray(opc, dtype=np.float64)
    if opc.ndim != 3 or opc.shape[0] < 2 or opc.shape[1] < 2:
        raise ValueError("organized cloud must be at least 2 x 2")
    M, N = opc.shape[:2]
    first, second = _quad_validity(opc)
    ok = np.empty((M - 1, N - 1, 2), dtype=bool)
    ok[..., 0] = first
    ok[..., 1] = second
    ok = ok.reshape(-1)
    trimap = np.full(ok.size, -1, dtype=np.int64)
    trimap[ok] = np.arange(int(ok.sum()), dtype=np.int64)

    u, v = np.meshgrid(np.arange(M - 1, dtype=np.int64),
                       np.arange(N - 1, dtype=np.int64), indexing="ij")
    i1 = u * N + v              # p1 = (u, v)
    i2 = i1 + 1                 # p2 = (u, v+1)
    i4 = i1 + N                 # p4 = (u+1, v)
    i3 = i4 + 1                 # p3 = (u+1, v+1)
    fc = np.empty((M - 1, N - 1, 2, 3), dtype=np.int64)
    fc[..., 0, :] = np.stack([i3, i2, i1], axis=-1)
    fc[..., 1, :] = np.stack([i1, i4, i3], axis=-1)
    return fc.reshape(-1, 3)[ok], trimap


def extract_halfedges_opc(trimap, M, N):
    """Twin half-edges of the OPC mesh: mesh.py:99-135.

    Edge k of a triangle always twins edge k of the neighbour:
      first (u,v,0):  e0 -> (u, v+1, 1), e1 -> (u-1, v, 1), e2 -> (u, v, 1)
      second (u,v,1): e0 -> (u, v-1, 0), e1 -> (u+1, v, 0), e2 -> (u, v, 0)
    he[3t+k] = 3*trimap[nbr]+k, or -1 off-grid / for an absent neighbour.
    """
    tm = np.asarray(trimap, dtype=np.int64).reshape(M - 1, N - 1, 2)
    n_tri = int(tm.max()) + 1 if tm.size else 0
    he = np.full(3 * max(n_tri, 0), -1, dtype=np.int64)
    Mq, Nq = M - 1, N - 1

    def shifted(plane, du, dv):
        out = np.full((Mq, Nq), -1, dtype=np.int64)
        su = slice(max(0, -du), min(Mq, Mq - du))
        sv = slice(max(0, -dv), min(Nq, Nq - dv))
        tu = slice(su.start + du, su.stop + du)
        tv = slice(sv.start + dv, sv.stop + dv)
        out[su, sv] = plane[tu, tv]
        return out

    first, second = tm[..., 0], tm[..., 1]
    links = (
        (first, 0, shifted(second, 0, 1)),
        (first, 1, shifted(second, -1, 0)),
        (first, 2, second),
        (second, 0, shifted(first, 0, -1)),
        (second, 1, shifted(first, 1, 0)),
        (second, 2, first),
    )
    for owner, k, target in links:
        m = (owner >= 0) & (target >= 0)
        he[3 * owner[m] + k] = 3 * target[m] + k
    return he


# ---------------------------------------------------------------------- normals
def _cross_unit(a, b, c):
    """cross(b-a, c-a)/|.|, NaN unless |.| > 0: geometry.py:134-147.

    Operation order reproduces numpy's np.cross / np.linalg.norm bit for bit:
    x = e1y*e2z - e1z*e2y, y = e1z*e2x - e1x*e2z, z = e1x*e2y - e1y*e2x,
    norm = sqrt((x*x + y*y) + z*z).
    """
    e1 = b - a
    e2 = c - a
    x = e1[..., 1] * e2[..., 2] - e1[..., 2] * e2[..., 1]
    y = e1[..., 2] * e2[..., 0] - e1[..., 0] * e2[..., 2]
    z = e1[..., 0] * e2[..., 1] - e1[..., 1] * e2[..., 0]
    nrm = np.sqrt((x * x + y * y) + z * z)
    out = np.stack([x, y, z], axis=-1)
    with np.errstate(invalid="ignore", divide="ignore"):
        out = out / nrm[..., None]
    out[~(nrm > 0.0)] = np.nan
    return out


def triangle_normals(points, triangles):
    """Per-triangle unit normals of an indexed set: geometry.py:134-147."""
    pts = np.asarray(points, dtype=np.float64)
    tri = np.asarray(triangles, dtype=np.int64)
    return _cross_unit(pts[tri[:, 0]], pts[tri[:, 1]], pts[tri[:, 2]])


def compute_fc_triangle_data(opc):
    """Centroids and normals of the fully-connected grid: smoothing.py:61-88.

    Shapes (M-1, N-1, 2, 3); centroid = ((a+b)+c)/3.0 with (a,b,c) =
    (p3,p2,p1) for k=0 and (p1,p4,p3) for k=1.
    """
    opc = np.asarray(opc, dtype=np.float64)
    if opc.ndim != 3 or opc.shape[0] < 2 or opc.shape[1] < 2:
        raise ValueError("organized cloud must be at least 2 x 2")
    p1, p2 = opc[:-1, :-1], opc[:-1, 1:]
    p3, p4 = opc[1:, 1:], opc[1:, :-1]
    Mq, Nq = p1.shape[:2]
    cen = np.empty((Mq, Nq, 2, 3))
    nrm = np.empty((Mq, Nq, 2, 3))
    for k, (a, b, c) in ((0, (p3, p2, p1)), (1, (p1, p4, p3))):
        cen[:, :, k] = ((a + b) + c) / 3.0
        nrm[:, :, k] = _cross_unit(a, b, c)
    return cen, nrm


# -------------------------------------------------------------------- bilateral
def bilateral_iterate(centroids, normals, sigma_length, sigma_angle,
                      kernel_size, iterations):
    """Bilateral normal filter on the FC triangle grid: _fallback.py:120-166.

    Neighbours: every triangle (u+du, v+dv, kk) of the (2h+1)^2 quad window
    (du, dv, kk loop order), self excluded, off-grid and non-finite-weight
    neighbours skipped; w = exp(-|dc|^2/(2 sl^2) - |dn|^2/(2 sa^2)); the new
    normal is acc/|acc| if wsum > 0 and |acc| > 1e-30, else unchanged.  NaN
    normals stay NaN.  Centroids never change.
    """
    C = np.asarray(centroids, dtype=np.float64)
    cur = np.array(normals, dtype=np.float64, copy=True)
    Mq, Nq = cur.shape[:2]
    h = kernel_size // 2
    a_c = 1.0 / (2.0 * sigma_length * sigma_length)
    a_n = 1.0 / (2.0 * sigma_angle * sigma_angle)
    for _ in range(iterations):
        acc = np.zeros_like(cur)
        wsum = np.zeros((Mq, Nq, 2))
        for du in range(-h, h + 1):
            for dv in range(-h, h + 1):
                u_lo, u_hi = max(0, -du), min(Mq, Mq - du)
                v_lo, v_hi = max(0, -dv), min(Nq, Nq - dv)
                if u_lo >= u_hi or v_lo >= v_hi:
                    continue
                dst = (slice(u_lo, u_hi), slice(v_lo, v_hi))
                src = (slice(u_lo + du, u_hi + du), slice(v_lo + dv, v_hi + dv))
                for kk in (0, 1):
                    nb_n = cur[src][:, :, kk]
                    nb_c = C[src][:, :, kk]
                    for k in (0, 1):
                        if du == 0 and dv == 0 and kk == k:
                            continue
                        dc = nb_c - C[dst][:, :, k]
                        dn = nb_n - cur[dst][:, :, k]
                        dc2 = dc[..., 0] ** 2 + dc[..., 1] ** 2 + dc[..., 2] ** 2
                        dn2 = dn[..., 0] ** 2 + dn[..., 1] ** 2 + dn[..., 2] ** 2
                        with np.errstate(invalid="ignore", over="ignore"):
                            w = np.exp(-dc2 * a_c - dn2 * a_n)
                        use = np.isfinite(w)
                        w = np.where(use, w, 0.0)
                        acc[dst + (k,)] += np.where(use[..., None], nb_n, 0.0) * w[..., None]
                        wsum[dst + (k,)] += w
        norm = np.sqrt(acc[..., 0] ** 2 + acc[..., 1] ** 2 + acc[..., 2] ** 2)
        upd = (wsum > 0.0) & (norm > 1e-30) & np.isfinite(cur).all(axis=3)
        nxt = cur.copy()
        nxt[upd] = acc[upd] / norm[upd][:, None]
        cur = nxt
    return cur


def bilateral_filter_opc(opc, sigma_length, sigma_angle, kernel_size,
                         iterations, trimap=None):
    """FC data -> bilateral -> gather to mesh order: smoothing.py:91-114."""
    opc = np.asarray(opc, dtype=np.float64)
    cen, nrm = compute_fc_triangle_data(opc)
    sm = bilateral_iterate(cen, nrm, sigma_length, sigma_angle, kernel_size, iterations)
    if trimap is None:
        _, trimap = extract_triangles_opc(opc)
    trimap = np.asarray(trimap, dtype=np.int64)
    sel = trimap >= 0
    out = np.empty((int(sel.sum()), 3))
    out[trimap[sel]] = sm.reshape(-1, 3)[sel]
    return out


# ------------------------------------------------------------------------ mesh
def mesh_from_opc(opc):
    """(points, triangles, halfedges, normals, trimap): mesh.py:167-180."""
    opc = np.asarray(opc, dtype=np.float64)
    tris, trimap = extract_triangles_opc(opc)
    he = extract_halfedges_opc(trimap, opc.shape[0], opc.shape[1])
    pts = opc.reshape(-1, 3)
    return dict(points=pts, triangles=tris, halfedges=he,
                normals=triangle_normals(pts, tris), trimap=trimap,
                grid_shape=opc.shape[:2])


def max_edge_mask(points, triangles, l_max):
    """True where the longest edge exceeds l_max: segmentation.py:59-67,73.

    edge lengths via sqrt((dx^2+dy^2)+dz^2) (np.linalg.norm, f64) of b-a, c-b,
    a-c; longest = max(|b-a|, max(|c-b|, |a-c|)).
    """
    pts = np.asarray(points, dtype=np.float64)
    tri = np.asarray(triangles, dtype=np.int64)
    a, b, c = pts[tri[:, 0]], pts[tri[:, 1]], pts[tri[:, 2]]

    def length(d):
        return np.sqrt((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2])

    longest = np.maximum(length(b - a), np.maximum(length(c - b), length(a - c)))
    return longest > l_max


def group_assignment(points, triangles, normals, dominant_normals, l_max, ang_min):
    """Per-triangle group labels (uint8): segmentation.py:52-74.

    argmax over n . d (numpy matmul, first maximum; NaN maximal), 255 unless the best
    score >= ang_min, 255 where the longest edge > l_max.
    """
    dn = np.atleast_2d(np.asarray(dominant_normals, dtype=np.float64))
    if not 1 <= len(dn) <= 254:
        raise ValueError(f"need 1..254 dominant normals, got {len(dn)}")
    sims = np.asarray(normals, dtype=np.float64) @ dn.T
    labels = np.argmax(sims, axis=1).astype(np.uint8)
    best = sims[np.arange(len(sims)), labels]
    labels[~(best >= ang_min)] = 255
    labels[max_edge_mask(points, triangles, l_max)] = 255
    return labels


def front_end(opc, laplacian=None, bilateral=None, l_max=None):
    """Organized branch of pipeline.run_scene: pipeline.py:125-134.

    ``laplacian`` = (lam, kernel_size, iterations) or None; ``bilateral`` =
    (sigma_length, sigma_angle, kernel_size, iterations) or None.  Returns
    the smoothed grid and the mesh dict (normals replaced by the bilateral
    result when it runs), plus the l_max mask when requested.
    """
    opc = np.asarray(opc, dtype=np.float64)
    if laplacian is not None:
        opc = laplacian_filter(opc, *laplacian)
    mesh = mesh_from_opc(opc)
    if bilateral is not None:
        mesh["normals"] = bilateral_filter_opc(opc, *bilateral, trimap=mesh["trimap"])
    if l_max is not None:
        mesh["lmax_mask"] = max_edge_mask(mesh["points"], mesh["triangles"], l_max)
    mesh["smoothed"] = opc
    return mesh


def grow_segment(triangles, halfedges, points, groups, visited, seed, label, anchor, normal,
                 ptp_max):
    """Region growing from one seed: _native.pyx:170-222 (explicit stack, the native
    backend's order; the member SET is order independent).  `visited` is updated in
    place; returns the sorted member indices."""
    tris = np.asarray(triangles, dtype=np.int64).reshape(-1, 3)
    he = np.asarray(halfedges, dtype=np.int64)
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    ax, ay, az = (float(x) for x in anchor)
    nx, ny, nz = (float(x) for x in normal)
    check = ptp_max > 0.0
    visited[seed] = 1
    stack, members = [int(seed)], [int(seed)]
    while stack:
        t = stack.pop()
        for e in range(3 * t, 3 * t + 3):
            tw = int(he[e])
            if tw < 0:
                continue
            c = tw // 3
            if groups[c] != label or visited[c]:
                continue
            if check:
                ok = True
                for k in range(3):
                    p = pts[tris[c, k]]
                    d = (p[0] - ax) * nx + (p[1] - ay) * ny + (p[2] - az) * nz
                    if abs(d) > ptp_max:
                        ok = False
                        break
                if not ok:
                    continue
            visited[c] = 1
            stack.append(c)
            members.append(c)
    return np.sort(np.asarray(members, dtype=np.int64))


def grow_segments(points, triangles, halfedges, groups, label, dominant_normal, ptp_max,
                  tri_min):
    """The triangle_indices of region_growing_task's kept segments for one label
    (segmentation.py:117-151): seeds ascending, anchor = seed centroid (numpy mean),
    kept when >= tri_min triangles."""
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    tris = np.asarray(triangles, dtype=np.int64).reshape(-1, 3)
    groups = np.asarray(groups)
    visited = np.zeros(len(tris), dtype=np.uint8)
    dn = np.asarray(dominant_normal, dtype=np.float64)
    out = []
    for seed in np.nonzero(groups == label)[0]:
        if visited[seed]:
            continue
        anchor = pts[tris[seed]].mean(axis=0)
        m = grow_segment(tris, halfedges, pts, groups, visited, int(seed), int(groups[seed]),
                         anchor, dn, ptp_max)
        if len(m) >= tri_min:
            out.append(m)
    return out
