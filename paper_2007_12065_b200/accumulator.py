"""FastGA histogram integration on the GPU.

Reference: flatpoly/accumulator.py:136-173 and _kernels.find_cells
(_kernels/_fallback.py:14-44 == _native.pyx:120-167).  The accumulator STRUCTURE
(refined icosahedron, sorted s2 ids, 1-ring neighbours, regression window) is built
by the reference (``flatpoly.accumulator.build_accumulator``) or any object with the
same attributes; this module runs the per-normal search and the vote on the device:

* ``find_cell_indices(ga, normals)`` -- accumulator.py:136-149;
* ``integrate_normals(ga, normals, sample_pct)`` -- accumulator.py:157-173 (every
  round(1/sample_pct)-th normal, non-finite rows skipped, counts += votes; the votes
  are device atomics into the histogram).
Peak detection / clustering (scipy) stay on the host, outside the hot path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._device import Staged, ptr, stream


class DeviceAccumulator:
    """Device copy of a GaussianAccumulator's search structure (uploaded once)."""

    def __init__(self, ga, device=None):
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.ids = torch.from_numpy(np.ascontiguousarray(ga.s2ids, dtype=np.uint64)
                                    .view(np.int64)).to(dev)
        self.normals = torch.from_numpy(np.ascontiguousarray(ga.normals, dtype=np.float64)).to(dev)
        self.neighbors = torch.from_numpy(np.ascontiguousarray(ga.neighbors, dtype=np.int64)).to(dev)
        self.slope = float(ga.model_slope)
        self.intercept = float(ga.model_intercept)
        self.window = (int(ga.window_lo), int(ga.window_hi))
        self.n_cells = len(ga.s2ids)

    def search(self, queries: torch.Tensor, stride: int = 1, counts: torch.Tensor | None = None,
               want_cells: bool = True):
        q = queries.reshape(-1, 3).contiguous().to(torch.float64)
        n = (q.shape[0] + stride - 1) // stride
        cells = torch.empty((n,), dtype=torch.int64, device=q.device) if want_cells else None
        _lib.check(_lib.lib().opcfe_find_cells(q.data_ptr(), n, stride, self.ids.data_ptr(),
                                               self.normals.data_ptr(), self.neighbors.data_ptr(),
                                               self.n_cells, self.slope, self.intercept,
                                               self.window[0], self.window[1], ptr(cells),
                                               ptr(counts), stream()),
                   "find_cells")
        return cells


def _device_acc(ga):
    cached = getattr(ga, "_opcfe_device", None)
    if cached is None:
        cached = DeviceAccumulator(ga)
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
    ga.counts = np.asarray(ga.counts) + counts.cpu().numpy()
    return ga.counts
