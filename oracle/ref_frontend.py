"""The REFERENCE's own CPU front-end, for the CPU baseline -- TEST/BENCH INFRASTRUCTURE ONLY.

Sequence of pipeline.run_scene's organized branch (pipeline.py:125-134):
    laplacian_filter_opc -> mesh_from_opc -> bilateral_filter_opc
with the reference's compiled kernels (oracle/_ref/_native.so, built by
oracle/build_ref.sh from /root/reference/pkg/src/flatpoly/_kernels/_native.pyx
with the reference's own flags) for the two hot loops -- laplacian_filter
(_native.pyx:225) and bilateral_iterate (_native.pyx:287) -- and the NumPy
restatement in flatpoly_oracle for the parts the reference itself runs in NumPy
(triangles / twins / normals / FC data / gather, mesh.py + smoothing.py).

If oracle/_ref is missing (reference not built), the C restatement
(oracle/opc_oracle.c) is used and the baseline is reported as kind "port".
Only bench.py's cpu_baseline / --impl reference legs call this.
"""

from __future__ import annotations

import importlib.util
import os
import time

import numpy as np

from . import flatpoly_oracle as fo

_HERE = os.path.dirname(os.path.abspath(__file__))
_NATIVE = None


def native():
    """The reference's compiled _native module, or None."""
    global _NATIVE
    if _NATIVE is None:
        so = os.path.join(_HERE, "_ref", "_native.so")
        if not os.path.exists(so):
            return None
        spec = importlib.util.spec_from_file_location("_native", so)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _NATIVE = mod
    return _NATIVE


def kind() -> str:
    return "reference" if native() is not None else "port"


def front_end(opc, lap=(1.0, 3, 10), bil=(0.1, 0.15, 3, 5)):
    """One frame through the reference's CPU implementation; returns stage timings (s)."""
    nat = native()
    t = {}
    t0 = time.perf_counter()
    opc = np.ascontiguousarray(opc, dtype=np.float64)
    if nat is not None:
        sm = nat.laplacian_filter(opc, float(lap[0]), int(lap[1]), int(lap[2])) if lap else opc
        t1 = time.perf_counter()
        tris, trimap = fo.extract_triangles_opc(sm)
        he = fo.extract_halfedges_opc(trimap, sm.shape[0], sm.shape[1])
        normals = fo.triangle_normals(sm.reshape(-1, 3), tris)
        t2 = time.perf_counter()
        if bil:
            cen, nrm = fo.compute_fc_triangle_data(sm)
            out = nat.bilateral_iterate(cen, nrm, float(bil[0]), float(bil[1]), int(bil[2]),
                                        int(bil[3]))
            sel = trimap >= 0
            normals = np.empty((int(sel.sum()), 3))
            normals[trimap[sel]] = out.reshape(-1, 3)[sel]
    else:
        from . import c_oracle
        sm = c_oracle.laplacian_filter(opc, *lap) if lap else opc
        t1 = time.perf_counter()
        tris, trimap, he = c_oracle.triangulate(sm)
        normals = c_oracle.triangle_normals(sm, tris)
        t2 = time.perf_counter()
        if bil:
            cen, nrm = c_oracle.compute_fc_triangle_data(sm)
            normals = c_oracle.gather(c_oracle.bilateral_iterate(cen, nrm, *bil), trimap, len(tris))
    t3 = time.perf_counter()
    t.update(laplacian=t1 - t0, front_end=t2 - t1, bilateral=t3 - t2, total=t3 - t0)
    return t, len(tris)


# ---------------------------------------------------------------- pool worker
_POOL_FRAME = None


def _init_worker(frame):
    global _POOL_FRAME
    os.environ["OMP_NUM_THREADS"] = "1"
    _POOL_FRAME = frame
    native()


def _work(args):
    row0, rows, lap, bil = args
    sub = _POOL_FRAME[row0:row0 + rows]
    t, _ = front_end(sub, lap, bil)
    return t["total"]


class ReferencePool:
    """Process pool running the reference front-end on row strips of one frame.

    The reference has no intra-frame parallelism (the _native.pyx loops are serial),
    so its best multi-core mode is one independent task per process.  A task is a
    horizontal strip of `rows` rows of the frame; a strip costs the same per pixel
    as the full frame (+ a 1-row overlap per strip, negligible), so a step of
    W strips of R rows credits W*R/M frames.
    """

    def __init__(self, frame, workers, rows, lap, bil):
        import multiprocessing as mp
        self.frame = frame
        self.workers = workers
        self.rows = rows
        self.lap, self.bil = lap, bil
        ctx = mp.get_context("fork")
        self.pool = ctx.Pool(workers, initializer=_init_worker, initargs=(frame,))

    def step(self):
        M = self.frame.shape[0]
        tasks = []
        for w in range(self.workers):
            row0 = (w * self.rows) % max(1, M - self.rows)
            tasks.append((row0, self.rows, self.lap, self.bil))
        t0 = time.perf_counter()
        self.pool.map(_work, tasks, chunksize=1)
        return time.perf_counter() - t0, self.workers * self.rows / M

    def close(self):
        self.pool.close()
        self.pool.join()
