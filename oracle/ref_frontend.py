"""The REFERENCE's own CPU front-end, timed for the CPU baseline -- BENCH INFRASTRUCTURE ONLY.

The stock code path: the unmodified reference package installed in baseline/_ref
(baseline/install_ref.sh: pip install of /root/reference/pkg, its Cython kernels built
by its own setup.py) running the organized branch of pipeline.run_scene
(pipeline.py:125-134) through its public API, one WHOLE frame per process:

    sm   = smoothing.laplacian_filter_opc(opc, LaplacianParams)         (smoothing.py:53)
    mesh = mesh.mesh_from_opc(sm)                                        (mesh.py:167)
    mesh.normals = smoothing.bilateral_filter_opc(sm, BilateralParams, mesh.trimap)

The reference has no intra-frame parallelism (its _native.pyx loops are serial), so its
best multi-core mode is one frame per process.  Math libraries
are single-threaded per process.

If baseline/_ref is missing, the reference's compiled kernels alone (oracle/_ref,
oracle/build_ref.sh) with the NumPy restatement around them are used ("reference-
kernels"), else the C restatement ("port").  Only bench.py's cpu_baseline /
--impl reference legs call this.
"""

from __future__ import annotations

import importlib.util
import os
import sys
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_REPO = os.path.dirname(_HERE)
REF_DIR = os.path.join(_REPO, "baseline", "_ref")
STUBS = os.path.join(_REPO, "tests", "golden", "_stubs")   # shapely import stub
_FLATPOLY = None
_NATIVE = None


def flatpoly():
    """The installed reference package (baseline/_ref), native backend, or None."""
    global _FLATPOLY
    if _FLATPOLY is None and os.path.isdir(os.path.join(REF_DIR, "flatpoly")):
        for p in (STUBS, REF_DIR):
            if p not in sys.path:
                sys.path.insert(0, p)
        os.environ.pop("FLATPOLY_PURE", None)
        os.environ.pop("FLATPOLY_CUDA", None)
        import flatpoly as fp
        import flatpoly.mesh  # noqa: F401
        import flatpoly.smoothing  # noqa: F401
        if fp.kernel_backend != "native":
            raise RuntimeError(f"baseline/_ref: kernel backend {fp.kernel_backend!r}, "
                               "expected the compiled 'native' one")
        _FLATPOLY = fp
    return _FLATPOLY


def native():
    """The reference's compiled _native module from oracle/_ref, or None."""
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
    if flatpoly() is not None:
        return "reference"
    return "reference" if native() is not None else "port"


def path_name() -> str:
    if flatpoly() is not None:
        return ("the stock reference (baseline/_ref flatpoly, native Cython backend): "
                "smoothing.laplacian_filter_opc -> mesh.mesh_from_opc -> "
                "smoothing.bilateral_filter_opc (pipeline.py:125-134)")
    if native() is not None:
        return ("the reference's compiled kernels (oracle/_ref) + NumPy restatement of "
                "mesh.py / smoothing.py (baseline/_ref missing)")
    return "the C restatement oracle/opc_oracle.c (reference not built)"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def front_end(opc, lap=(1.0, 3, 10), bil=(0.1, 0.15, 3, 5), want=False):
    """One frame through the reference; returns (stage timings in s, T, outputs or None)."""
    fp = flatpoly()
    t0 = time.perf_counter()
    opc = np.asarray(opc, dtype=np.float64)
    if fp is not None:
        from flatpoly.mesh import mesh_from_opc
        from flatpoly.smoothing import (BilateralParams, LaplacianParams, bilateral_filter_opc,
                                        laplacian_filter_opc)
        sm = laplacian_filter_opc(opc, LaplacianParams(*lap)) if lap else opc
        t1 = time.perf_counter()
        mesh = mesh_from_opc(sm)
        t2 = time.perf_counter()
        if bil:
            mesh.normals = bilateral_filter_opc(sm, BilateralParams(*bil), mesh.trimap)
        tris, trimap, he, normals = mesh.triangles, mesh.trimap, mesh.halfedges, mesh.normals
    elif native() is not None:
        from . import flatpoly_oracle as fo
        nat = native()
        sm = nat.laplacian_filter(np.ascontiguousarray(opc), float(lap[0]), int(lap[1]),
                                  int(lap[2])) if lap else opc
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
    t = dict(laplacian=t1 - t0, front_end=t2 - t1, bilateral=t3 - t2, total=t3 - t0)
    out = None
    if want:
        out = dict(smoothed=np.asarray(sm), trimap=np.asarray(trimap),
                   n_halfedges_linked=int((np.asarray(he) >= 0).sum()),
                   normals=np.asarray(normals))
    return t, len(tris), out


# ---------------------------------------------------------------- pool worker
_POOL_FRAME = None


def _init_worker(frame):
    global _POOL_FRAME
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"
    _POOL_FRAME = frame
    kind()                                  # import the reference once per process


def _work(args):
    frames, lap, bil, want = args
    total, outs = 0.0, None
    for i in range(frames):
        t, _, o = front_end(_POOL_FRAME, lap, bil, want=want and i == 0)
        total += t["total"]
        outs = outs or o
    return total, outs


class ReferencePool:
    """One process per host core, each running the reference on WHOLE frames."""

    def __init__(self, frame, workers, lap, bil, frames_per_task=1):
        import multiprocessing as mp
        self.frame = frame
        self.workers = workers
        self.lap, self.bil = lap, bil
        self.per_task = frames_per_task
        ctx = mp.get_context("fork")
        self.pool = ctx.Pool(workers, initializer=_init_worker, initargs=(frame,))

    def step(self, want_sample=False):
        """All workers run `frames_per_task` whole frames; -> (seconds, frames, sample)."""
        tasks = [(self.per_task, self.lap, self.bil, want_sample and w == 0)
                 for w in range(self.workers)]
        t0 = time.perf_counter()
        res = self.pool.map(_work, tasks, chunksize=1)
        dt = time.perf_counter() - t0
        return dt, self.workers * self.per_task, res[0][1]

    def close(self):
        self.pool.close()
        self.pool.join()
