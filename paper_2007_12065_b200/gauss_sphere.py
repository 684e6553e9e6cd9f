"""Host-side build of the FastGA accumulator STRUCTURE (one-time setup, NumPy).

What the GPU search (`accumulator.find_cell_indices` / `integrate_normals`, csrc/fastga.cu)
needs from a level-L Gaussian accumulator, bit-identical to the reference's
`build_accumulator(L)` (accumulator.py:76-133) so every cell index, vote and neighbour
row agrees:

* the refined icosahedron (icosphere.py:41-141): 12 base vertices (poles + two rings of
  five, the lower ring turned by pi/5), 20 faces in five strips of four; each refinement
  splits a face (a, b, c) into (a, ab, ac), (b, bc, ab), (c, ac, bc), (ab, bc, ac), with
  a midpoint created the first time its edge is met in (ab, bc, ac) face order and
  projected back onto the unit sphere;
* cell normals = normalised triangle centroids (icosphere.py:33-37);
* 64-bit cell ids (sfc.py:46-104): cube face of the dominant axis (chain -y, +x, +z,
  -x, -z, +y), tangent-warped face coordinates quantised to 30 bits, a per-face dihedral
  transform, and the Hilbert position of the cell -- computed here with a two-flag
  state machine (swap / complement of the remaining low bits) instead of rotating the
  coordinates level by level;
* cells sorted by id, the 1-ring neighbour matrix (icosphere.py:144-166: every other
  cell sharing a vertex, ascending, -1 padded to 12) re-indexed into sorted order, and
  the least-squares index model with its bracketing window (accumulator.py:84-101).

Vectorised over faces / cells; the only per-element Python loop is the vertex
normalisation, kept on the reference's own 1-D `np.linalg.norm` (a BLAS dot whose
rounding the vectorised forms do not reproduce).  Peak detection (unwrap layout,
vertex-cell incidence) is outside the hot path and not built.
"""

from __future__ import annotations

import functools

import numpy as np

MAX_LEVEL = 7
_BITS = 30                     # Hilbert order per face (sfc.py:16)
_GRID = 1 << _BITS

# Cube faces along the id chain, keyed by (dominant axis, negative?): the face index,
# the (u, v) axes of its plane, and the dihedral transform (swap u/v, complement u,
# complement v) that joins each face's curve exit to the next face's entry (sfc.py:20-35).
_FACE_TABLE = {
    (1, True): (0, 0, 2, False, False, False),
    (0, False): (1, 1, 2, True, False, False),
    (2, False): (2, 0, 1, False, True, False),
    (0, True): (3, 1, 2, True, True, False),
    (2, True): (4, 0, 1, True, False, False),
    (1, False): (5, 0, 2, False, False, False),
}


def _face_lookup():
    idx = np.zeros(6, dtype=np.int64)              # axis * 2 + negative -> face
    uax = np.zeros(6, dtype=np.int64)              # per face
    vax = np.zeros(6, dtype=np.int64)
    swp = np.zeros(6, dtype=bool)
    ngu = np.zeros(6, dtype=bool)
    ngv = np.zeros(6, dtype=bool)
    for (axis, neg), (face, u, v, s, nu, nv) in _FACE_TABLE.items():
        idx[axis * 2 + int(neg)] = face
        uax[face], vax[face], swp[face], ngu[face], ngv[face] = u, v, s, nu, nv
    return idx, uax, vax, swp, ngu, ngv


_FACE_OF, _U_AX, _V_AX, _SWAP, _NEG_U, _NEG_V = _face_lookup()


def hilbert_index(x: np.ndarray, y: np.ndarray, bits: int = _BITS) -> np.ndarray:
    """Hilbert-curve position of integer cells (x, y) in [0, 2^bits)^2.

    Same curve as the textbook xy -> d walk (quadrant digit (3 rx) ^ ry, then for ry = 0
    complement both coordinates if rx = 1 and swap them): that walk only ever swaps or
    complements the remaining low bits, and the two commute, so its whole history is two
    flags applied to the ORIGINAL bits of each level.
    """
    x = np.asarray(x, dtype=np.int64)
    y = np.asarray(y, dtype=np.int64)
    d = np.zeros(np.broadcast(x, y).shape, dtype=np.int64)
    swap = np.zeros(d.shape, dtype=bool)
    comp = np.zeros(d.shape, dtype=bool)
    for level in range(bits - 1, -1, -1):
        bx = ((x >> level) & 1).astype(bool)
        by = ((y >> level) & 1).astype(bool)
        rx = np.where(swap, by, bx) ^ comp
        ry = np.where(swap, bx, by) ^ comp
        d = (d << 2) | ((3 * rx.astype(np.int64)) ^ ry.astype(np.int64))
        turn = ~ry
        comp = comp ^ (turn & rx)
        swap = swap ^ turn
    return d


def _quantise(t: np.ndarray) -> np.ndarray:
    w = np.arctan(t) * (4.0 / np.pi)               # area-equalising tangent warp
    return np.clip(np.floor((w + 1.0) * 0.5 * _GRID).astype(np.int64), 0, _GRID - 1)


def s2_ids(normals: np.ndarray) -> np.ndarray:
    """uint64 ids of (n, 3) normals: face (3 bits) << 60 | 60-bit Hilbert position."""
    n = np.atleast_2d(np.asarray(normals, dtype=np.float64))
    norms = np.linalg.norm(n, axis=1)
    if not np.all(np.isfinite(norms)) or np.any(norms == 0.0):
        raise ValueError("normals must be finite and nonzero")
    n = n / norms[:, None]
    rows = np.arange(n.shape[0])
    axis = np.argmax(np.abs(n), axis=1)
    dom = n[rows, axis]
    face = _FACE_OF[axis * 2 + (dom < 0)]
    iu = _quantise(n[rows, _U_AX[face]] / np.abs(dom))
    iv = _quantise(n[rows, _V_AX[face]] / np.abs(dom))
    sw = _SWAP[face]
    iu, iv = np.where(sw, iv, iu), np.where(sw, iu, iv)
    iu = np.where(_NEG_U[face], _GRID - 1 - iu, iu)
    iv = np.where(_NEG_V[face], _GRID - 1 - iv, iv)
    return (face.astype(np.uint64) << np.uint64(2 * _BITS)) | \
        hilbert_index(iu, iv).astype(np.uint64)


def _base_icosahedron():
    h = 1.0 / np.sqrt(5.0)
    c = 2.0 / np.sqrt(5.0)
    verts = [np.array([0.0, 0.0, 1.0])]
    verts += [np.array([c * np.cos(2.0 * np.pi * i / 5.0), c * np.sin(2.0 * np.pi * i / 5.0), h])
              for i in range(5)]
    verts += [np.array([c * np.cos(2.0 * np.pi * i / 5.0 + np.pi / 5.0),
                        c * np.sin(2.0 * np.pi * i / 5.0 + np.pi / 5.0), -h]) for i in range(5)]
    verts.append(np.array([0.0, 0.0, -1.0]))
    s = np.arange(5)
    up, up1, lo, lo1 = 1 + s, 1 + (s + 1) % 5, 6 + s, 6 + (s + 1) % 5
    top, bot = np.zeros(5, np.int64), np.full(5, 11, np.int64)
    strip = np.stack([np.stack([top, up, up1], 1), np.stack([up, lo, up1], 1),
                      np.stack([up1, lo, lo1], 1), np.stack([lo, bot, lo1], 1)], 1)
    return np.array(verts), strip.reshape(20, 3).astype(np.int64)


def refined_icosahedron(level: int):
    """(vertices (10*4^L+2, 3), triangles (20*4^L, 3)) in the reference's order."""
    if not 0 <= level <= MAX_LEVEL:
        raise ValueError(f"refinement level must be in [0, {MAX_LEVEL}], got {level}")
    V, F = _base_icosahedron()
    for _ in range(level):
        a, b, c = F[:, 0], F[:, 1], F[:, 2]
        edges = np.stack([np.stack([a, b], 1), np.stack([b, c], 1), np.stack([a, c], 1)],
                         1).reshape(-1, 2)                      # request order: ab, bc, ac
        lo, hi = edges.min(1), edges.max(1)
        key = lo * len(V) + hi
        _, first, inv = np.unique(key, return_index=True, return_inverse=True)
        order = np.argsort(first)                               # first-request order
        rank = np.empty_like(order)
        rank[order] = np.arange(len(order))
        mid = (len(V) + rank[inv]).reshape(-1, 3)               # per face: ab, bc, ac
        P = V[lo[first[order]]] + V[hi[first[order]]]
        P = P / np.array([np.linalg.norm(p) for p in P])[:, None]
        V = np.concatenate([V, P])
        ab, bc, ac = mid[:, 0], mid[:, 1], mid[:, 2]
        F = np.stack([np.stack([a, ab, ac], 1), np.stack([b, bc, ab], 1),
                      np.stack([c, ac, bc], 1), np.stack([ab, bc, ac], 1)], 1).reshape(-1, 3)
    return V, F


def cell_normals(V: np.ndarray, F: np.ndarray) -> np.ndarray:
    cen = V[F].mean(axis=1)
    return cen / np.linalg.norm(cen, axis=1)[:, None]


def one_ring(F: np.ndarray, nv: int) -> np.ndarray:
    """(nt, 12) ascending indices of the other cells sharing a vertex, -1 padded."""
    nt = len(F)
    flat = F.reshape(-1)
    by_vertex = np.argsort(flat, kind="stable")
    count = np.bincount(flat, minlength=nv)
    start = np.concatenate([[0], np.cumsum(count)[:-1]])
    width = int(count.max())
    slot = np.arange(len(flat)) - np.repeat(start, count)
    inc = np.full((nv, width), -1, dtype=np.int64)
    inc[flat[by_vertex], slot] = by_vertex // 3                 # incident triangles
    cand = inc[F].reshape(nt, -1)
    big = np.int64(nt)
    cand = np.where((cand < 0) | (cand == np.arange(nt)[:, None]), big, cand)
    cand.sort(axis=1)
    dup = np.zeros_like(cand, dtype=bool)
    dup[:, 1:] = cand[:, 1:] == cand[:, :-1]
    cand[dup] = big
    cand.sort(axis=1)
    if (cand[:, 12:] != big).any():
        raise RuntimeError("a cell has more than 12 one-ring neighbours")
    return np.where(cand[:, :12] == big, -1, cand[:, :12])


@functools.lru_cache(maxsize=None)
def accumulator_structure(level: int):
    """(normals, s2ids, neighbours, slope, intercept, window_lo, window_hi), cells sorted
    by id; arrays read-only (cached per level, like accumulator.py:76)."""
    V, F = refined_icosahedron(level)
    cells = cell_normals(V, F)
    ids = s2_ids(cells)
    order = np.argsort(ids, kind="stable")
    ids_sorted = ids[order]
    if np.any(ids_sorted[1:] == ids_sorted[:-1]):
        raise RuntimeError("space-filling-curve ids collided; refinement too deep")
    inv = np.empty(len(order), dtype=np.int64)
    inv[order] = np.arange(len(order))
    ring = one_ring(F, len(V))[order]
    nbrs = np.where(ring >= 0, inv[np.maximum(ring, 0)], -1)
    # least-squares line index ~ id and the error bounds of the search window
    idx = np.arange(len(ids_sorted), dtype=np.float64)
    x = ids_sorted.astype(np.float64)
    xm = x.mean()
    slope = ((x - xm) @ (idx - idx.mean())) / ((x - xm) @ (x - xm))
    intercept = idx.mean() - slope * xm
    err = idx - (slope * x + intercept)
    lo, hi = int(np.floor(err.min())) - 1, int(np.ceil(err.max())) + 1
    normals = np.ascontiguousarray(cells[order])
    for arr in (normals, ids_sorted, nbrs):
        arr.setflags(write=False)
    return normals, ids_sorted, nbrs, float(slope), float(intercept), lo, hi
