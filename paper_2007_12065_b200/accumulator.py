"""FastGA histogram integration on the GPU.

Reference: flatpoly/accumulator.py:76-173 and _kernels.find_cells
(_kernels/_fallback.py:14-44 == _native.pyx:120-167).

* ``build_accumulator(level)`` -- accumulator.py:104-133: the accumulator STRUCTURE
  (refined icosahedron, sorted s2 ids, 1-ring neighbours, regression window), built once
  per level on the host by ``gauss_sphere`` (vectorised NumPy, bit-identical to the
  reference's at every level 0..7); counts start at zero.  A reference-built
  ``GaussianAccumulator`` (or any object with the same attributes) works too;
* ``find_cell_indices(ga, normals)`` / ``find_cell_index`` -- accumulator.py:136-154;
* ``integrate_normals(ga, normals, sample_pct)`` -- accumulator.py:157-173 (every
  round(1/sample_pct)-th normal, non-finite rows skipped, counts += votes; the votes
  are device atomics into the histogram).
Peak detection / clustering (unwrap, scipy) stay outside the hot path and are not built.
"""

from __future__ import annotations

import numpy as np
import torch

from dataclasses import dataclass

from . import _lib, gauss_sphere
from ._device import Staged, ptr, stream

MAX_LEVEL = gauss_sphere.MAX_LEVEL


@dataclass
class GaussianAccumulator:
    """Histogram cells sorted by s2 id plus the search structures (accumulator.py:35-58,
    without the peak-detection fields)."""

    level: int
    normals: np.ndarray        # (n, 3) cell normals, sorted by id
    s2ids: np.ndarray          # (n,) uint64, strictly ascending
    neighbors: np.ndarray      # (n, 12) cell indices, -1 padded
    model_slope: float
    model_intercept: float
    window_lo: int
    window_hi: int
    counts: np.ndarray         # (n,) int64 votes

    @property
    def num_cells(self) -> int:
        return len(self.s2ids)


def build_accumulator(level: int) -> GaussianAccumulator:
    """A level-``level`` accumulator with zero counts (accumulator.py:104-133); the
    structure is built once per level and shared (read-only)."""
    if not 0 <= level <= MAX_LEVEL:
        raise ValueError(f"level must be in [0, {MAX_LEVEL}], got {level}")
    normals, ids, nbrs, slope, intercept, lo, hi = gauss_sphere.accumulator_structure(level)
    return GaussianAccumulator(level=level, normals=normals, s2ids=ids, neighbors=nbrs,
                               model_slope=slope, model_intercept=intercept, window_lo=lo,
                               window_hi=hi, counts=np.zeros(len(ids), dtype=np.int64))


class DeviceAccumulator:
    """Device copy of a GaussianAccumulator's search structure (uploaded once)."""

    def __init__(self, ga, device=None):
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device

        def up(a, dtype):   # a host copy first: the shared structures are read-only
            return torch.from_numpy(np.array(a, dtype=dtype, order="C", copy=True)).to(dev)
        self.ids = up(np.ascontiguousarray(ga.s2ids, dtype=np.uint64).view(np.int64), np.int64)
        self.normals = up(ga.normals, np.float64)
        self.neighbors = up(ga.neighbors, np.int64)
        self.slope = float(ga.model_slope)
        self.intercept = float(ga.model_intercept)
        self.window = (int(ga.window_lo), int(ga.window_hi))
        self.n_cells = len(ga.s2ids)

    def search(self, queries: torch.Tensor, stride: int = 1, counts: torch.Tensor | None = None,
               want_cells: bool = True):
        q = queries.reshape(-1, 3).contiguous().to(torch.float64)
        n = (q.shape[0] + stride - 1) // stride
        cells = torch.empty((n,), dtype=torch.int64, device=q.device) if want_cells else None
        if n == 0:
            return cells
        _lib.check(_lib.lib().opcfe_find_cells(q.data_ptr(), n, stride, self.ids.data_ptr(),
                                               self.normals.data_ptr(), self.neighbors.data_ptr(),
                                               self.n_cells, self.slope, self.intercept,
                                               self.window[0], self.window[1], ptr(cells),
                                               ptr(counts), stream()),
                   "find_cells")
        return cells


_LEVEL_DEVICE = {}   # (level, device) -> the device copy of a build_accumulator structure


def _device_acc(ga):
    cached = getattr(ga, "_opcfe_device", None)
    if cached is None:
        key = None
        if isinstance(ga, GaussianAccumulator) and 0 <= ga.level <= MAX_LEVEL and \
                ga.s2ids is gauss_sphere.accumulator_structure(ga.level)[1]:
            key = (ga.level, torch.cuda.current_device())   # shared, read-only structure
            cached = _LEVEL_DEVICE.get(key)
        if cached is None:
            cached = DeviceAccumulator(ga)
            if key is not None:
                _LEVEL_DEVICE[key] = cached
        try:
            ga._opcfe_device = cached
        except AttributeError:
            pass
    return cached


def find_cell_indices(ga, normals):
    """Vectorized cell lookup for an (n, 3) array of unit normals (accumulator.py:136-149)."""
    S = Staged(normals)
    q = S.dev.reshape(-1, 3).to(torch.float64)
    sq = (q * q).sum(dim=1)
    if not bool(torch.isfinite(sq).all()) or bool((sq == 0).any()):
        raise ValueError("query normals must be finite and nonzero")
    return S.give(_device_acc(ga).search(q))


def find_cell_index(ga, normal) -> int:
    """Cell index whose normal is (near-)closest to ``normal`` (accumulator.py:152-154)."""
    return int(find_cell_indices(ga, np.asarray(normal, dtype=np.float64)[None, :])[0])


def integrate_normals(ga, normals, sample_pct: float = 1.0):
    """Vote every round(1/sample_pct)-th normal into ga.counts (accumulator.py:157-173)."""
    if not 0.0 < sample_pct <= 1.0:
        raise ValueError("sample_pct must be in (0, 1]")
    S = Staged(normals)
    q = S.dev.reshape(-1, 3).to(torch.float64).contiguous()
    stride = max(1, int(round(1.0 / sample_pct)))
    acc = _device_acc(ga)
    counts = torch.zeros((acc.n_cells,), dtype=torch.int64, device=q.device)
    acc.search(q, stride=stride, counts=counts, want_cells=False)
    votes = counts.cpu().numpy()
    cur = ga.counts
    if isinstance(cur, np.ndarray) and cur.flags.writeable and cur.dtype == np.int64:
        cur += votes                                   # in place, like accumulator.py:172
    else:
        ga.counts = np.asarray(cur) + votes
    return ga.counts
