"""The organized front-end as one device-resident engine (reference: the organized
branch of flatpoly.pipeline.run_scene, pipeline.py:125-134).

    laplacian_filter_opc -> mesh_from_opc -> bilateral_filter_opc (-> l_max mask)

``FrontEnd`` owns every buffer for a batch of F frames of M x N points, launches
the whole chain through ONE C-ABI call (``opcfe_front_end``) and, by default,
replays it as a CUDA graph (one graph launch per batch instead of ~2 + L + B
kernel launches).  Frames are independent: a batch is the unit of work of one
GPU, and multi-GPU runs shard batches over ranks without any collective.

Host path (``run_host``): pinned host input -> H2D -> graph -> D2H of every mesh
output into pinned host buffers, the three phases overlapped across frames on
separate streams.
"""

from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._device import host_view, points_pitch, require_cuda
from .mesh import HalfEdgeMesh
from .smoothing import BilateralParams, LaplacianParams


def _lap_from32(N: int, src_kind: int, kernel_size: int) -> bool:
    """Whether a strict / mixed front end smooths an fp32 source without the conversion
    pass (csrc/strict.cu laplacian64_from32_ok: k = 3, even N, 16-B source rows; the
    front end's own buffers are 16-B aligned)."""
    on = os.environ.get("OPCFE_LAP64_FROM32", "1")[:1] != "0" and \
        os.environ.get("OPCFE_LAP64_TMA", "1")[:1] != "0"
    rows16 = src_kind == 0 or (3 * N) % 4 == 0                # padded grids: pitch % 4 == 0
    return on and src_kind != 2 and kernel_size == 3 and N % 2 == 0 and rows16


def _lap_mask_fused(N: int, kernel_size: int) -> bool:
    """Whether the strict / mixed Laplacian's first pass writes the validity bits itself
    (csrc/strict.cu laplacian64_mask_fused: the TMA kernels, k = 3, even N)."""
    return os.environ.get("OPCFE_LAP64_TMA", "1")[:1] != "0" and kernel_size == 3 and N % 2 == 0


def _mixed_fc_fused(N: int, iterations: int) -> bool:
    """Whether the mixed front end computes its FC data inside the fused bilateral
    iteration 1 (csrc/bilateral.cu bilateral_fc_in_iteration1): even N, >= 2 iterations."""
    on = os.environ.get("OPCFE_MIXED_FUSED_FC", "1")[:1] != "0" and \
        os.environ.get("OPCFE_BILATERAL_PACKED", "1")[:1] != "0"
    return on and N % 2 == 0 and iterations >= 2


@dataclass
class FrontEndResult:
    """Device (or pinned host) outputs of one batch; rows beyond n_tri[f] are unused.
    Float outputs are fp32 (precision "fast") or float64 ("strict", "mixed")."""
    points: torch.Tensor        # (F, M, N, 3) smoothed grid (fast: view of the padded buffer)
    triangles: torch.Tensor     # (F, G, 3) int64, GID order
    trimap: torch.Tensor        # (F, G) int64
    halfedges: torch.Tensor     # (F, 3G) int64 or None
    normals: torch.Tensor       # (F, G, 3) (bilateral result, or triangle normals)
    lmax_mask: torch.Tensor     # (F, G) uint8 or None
    n_tri: list = field(default_factory=list)
    grid_shape: tuple = None
    labels: torch.Tensor = None  # (F, G) uint8 group labels (255 = unassigned) or None

    def mesh(self, f: int = 0) -> HalfEdgeMesh:
        """Frame f as a HalfEdgeMesh (flatpoly.mesh.HalfEdgeMesh fields)."""
        T = int(self.n_tri[f])
        return HalfEdgeMesh(
            points=self.points[f].reshape(-1, 3),
            triangles=self.triangles[f, :T],
            halfedges=None if self.halfedges is None else self.halfedges[f, :3 * T],
            normals=None if self.normals is None else self.normals[f, :T],
            trimap=self.trimap[f],
            grid_shape=self.grid_shape,
        )


class FrontEnd:
    """Batched organized front-end engine on one GPU.

    precision "fast" (default): fp32 kernels (+ the fp64 steps of the 1e-5 contract);
    "strict": the reference's own fp64 chain (opcfe_front_end with
    OPCFE_PRECISION_STRICT) -- float64 points and normals, bit-exact Laplacian and
    topology, bilateral normals within a few ulp of the reference chain;
    "mixed": a float64 Laplacian with rsqrt pair weights (vertices within a few ulp of
    the reference's), exact topology and FC data, then the fp32 bilateral
    on the FC arrays (OPCFE_PRECISION_MIXED) -- float64 outputs, normals within 1e-5 of the
    reference chain end to end on the benchmark frames.
    """

    def __init__(self, M: int, N: int, frames: int = 1,
                 laplacian: LaplacianParams | None = LaplacianParams(),
                 bilateral: BilateralParams | None = BilateralParams(),
                 l_max: float | None = None, halfedges: bool = True, normals: bool = True,
                 dominant_normals=None, ang_min: float = 0.95,
                 src_dtype=torch.float32, device=None, graph: bool = True,
                 precision: str = "fast", index_dtype=torch.int64):
        require_cuda()
        if index_dtype not in (torch.int64, torch.int32):
            raise ValueError("index_dtype must be torch.int64 (reference) or torch.int32")
        if precision not in ("fast", "strict", "mixed"):
            raise ValueError(f"precision must be 'fast', 'strict' or 'mixed', got {precision!r}")
        self.precision = precision
        self.strict = precision == "strict"
        self.f64 = f64 = precision in ("strict", "mixed")   # float64 grid / normals outputs
        if M < 2 or N < 2:
            from .geometry import DegenerateInputError
            raise DegenerateInputError("organized cloud must be at least 2 x 2")
        if laplacian is not None and min(M, N) < laplacian.kernel_size:
            from .geometry import DegenerateInputError
            raise DegenerateInputError("grid smaller than the filter kernel")
        self.M, self.N, self.F = M, N, frames
        self.device = (torch.device("cuda", torch.cuda.current_device()) if device is None
                       else torch.device(device))
        dev = self.device
        self.G = G = 2 * (M - 1) * (N - 1)
        self.pitch = points_pitch(N)
        self.src = torch.empty((frames, M, N, 3), dtype=src_dtype, device=dev)
        if src_dtype == torch.float32 and 3 * N == self.pitch:
            src_kind, src_pitch = 0, self.pitch
        else:
            src_kind, src_pitch = (2 if src_dtype == torch.float64 else 1), 0
        self.p = _lib.FrontEndParams(
            laplacian.iterations if laplacian else 0, laplacian.kernel_size if laplacian else 3,
            laplacian.lam if laplacian else 1.0,
            bilateral.iterations if bilateral else 0, bilateral.kernel_size if bilateral else 3,
            bilateral.sigma_length if bilateral else 0.1, bilateral.sigma_angle if bilateral else 0.15,
            float(l_max) if l_max is not None else -1.0)
        self.p.precision = {"fast": _lib.PRECISION_FAST, "strict": _lib.PRECISION_STRICT,
                            "mixed": _lib.PRECISION_MIXED}[precision]
        self.dn = None
        if dominant_normals is not None:   # fused group_assignment (segmentation.py:52-74)
            dn = torch.as_tensor(np.atleast_2d(np.asarray(dominant_normals, dtype=np.float64)))
            if not 1 <= dn.shape[0] <= 254:
                raise ValueError(f"need 1..254 dominant normals, got {dn.shape[0]}")
            self.dn = dn.to(dev).contiguous()
            self.p.dominant_normals = self.dn.data_ptr()
            self.p.n_dominant = self.dn.shape[0]
            self.p.ang_min = float(ang_min)
        fdt = torch.float64 if f64 else torch.float32
        self.grid = torch.empty((frames, M, N, 3) if f64 else (frames, M, self.pitch),
                                dtype=fdt, device=dev)
        self.trimap = torch.empty((frames, G), dtype=torch.int64, device=dev)
        self.triangles = torch.empty((frames, G, 3), dtype=torch.int64, device=dev)
        self.halfedges = torch.empty((frames, 3 * G), dtype=torch.int64, device=dev) if halfedges else None
        self.normals = torch.empty((frames, G, 3), dtype=fdt, device=dev) if normals else None
        self.lmax = torch.empty((frames, G), dtype=torch.uint8, device=dev) if l_max is not None else None
        self.n_tri = torch.empty((frames,), dtype=torch.int64, device=dev)
        self.labels = torch.empty((frames, G), dtype=torch.uint8, device=dev) \
            if self.dn is not None else None
        L = _lib.lib()
        ws_bytes = int(L.opcfe_front_end_workspace(frames, M, N, ctypes.byref(self.p), src_kind,
                                                   src_pitch))
        self.ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        self.io = _lib.FrontEndIO(
            self.src.data_ptr(), src_kind, src_pitch, self.grid.data_ptr(), self.trimap.data_ptr(),
            self.triangles.data_ptr(),
            self.halfedges.data_ptr() if halfedges else None,
            self.normals.data_ptr() if normals else None,
            self.lmax.data_ptr() if self.lmax is not None else None,
            self.n_tri.data_ptr(),
            self.labels.data_ptr() if self.labels is not None else None)
        # compact (NON-reference) int32 copies of the index outputs, narrowed on the device
        # after the chain (opcfe_narrow_indices) so that half the bytes cross PCIe
        self.index_dtype = index_dtype
        self.trimap32 = self.triangles32 = self.halfedges32 = None
        if index_dtype == torch.int32:
            if M * N >= 2 ** 31 or 3 * G >= 2 ** 31:
                raise ValueError("int32 indices need M*N and 6(M-1)(N-1) below 2^31")
            self.trimap32 = torch.empty((frames, G), dtype=torch.int32, device=dev)
            self.triangles32 = torch.empty((frames, G, 3), dtype=torch.int32, device=dev)
            self.halfedges32 = torch.empty((frames, 3 * G), dtype=torch.int32, device=dev) \
                if halfedges else None
        self._graph = None
        self._use_graph = graph
        extras = (normals and bilateral is None) or l_max is not None
        self.kernel_launches = self._count_launches(laplacian, bilateral if normals else None,
                                                    src_kind, extras, precision, N) + \
            (1 if self.labels is not None else 0) + \
            (0 if self.trimap32 is None else (3 if halfedges else 2))

    @staticmethod
    def _count_launches(lap, bil, src_kind, extras=False, precision="fast", N=0):
        """Kernels one batch launches (mirrors front_end_impl in csrc/capi.cu)."""
        from .smoothing import BILATERAL_MAX_K32, LAPLACIAN_MAX_K32
        strict, f64 = precision == "strict", precision in ("strict", "mixed")
        lap64 = lap is not None and (f64 or lap.kernel_size > LAPLACIAN_MAX_K32)
        bil64 = bil is not None and (strict or bil.kernel_size > BILATERAL_MAX_K32)
        n = 3                                                   # triangulate: count, scan, emit
        if f64 or lap64:
            from32 = f64 and lap is not None and _lap_from32(N, src_kind, lap.kernel_size)
            n += 1 if (src_kind != 2 and not from32) else 0     # source -> f64 (unstage)
            n += lap.iterations if lap else 0                   # laplacian_f64
            mask_fused = f64 and lap is not None and _lap_mask_fused(N, lap.kernel_size)
            n += 1 if (lap or f64) and not mask_fused else 0    # validity bits (+ fp32 grid)
            n += 1 if (f64 and extras) else 0                   # tri_extras_f64
        else:
            n += lap.iterations if lap else 0
            if not lap or src_kind != 0:
                n += 1                                          # stage-in
        if not f64:
            n += 1 if extras else 0                             # quad_extras: normals / l_max
        if bil64:
            n += 0 if (f64 or lap64) else 1                     # fp32 grid -> f64 (unstage)
            n += 1 + bil.iterations                             # fc_data_f64 + bilateral_f64
        elif bil and f64:                                       # mixed: fc_mixed + fp32
            n += bil.iterations                                 # iterations (f64 scatter);
            n += 0 if _mixed_fc_fused(N, bil.iterations) else 1  # FC data in iteration 1
        elif bil:
            n += bil.iterations
        return n

    # ------------------------------------------------------------------ device
    def _launch(self, stream: torch.cuda.Stream):
        L = _lib.lib()
        rc = L.opcfe_front_end(self.F, self.M, self.N, ctypes.byref(self.p),
                               ctypes.byref(self.io), self.ws.data_ptr(), self.ws.numel(),
                               stream.cuda_stream)
        _lib.check(rc, "front_end")
        self._narrow(stream)

    def _narrow(self, stream):
        if self.trimap32 is None:
            return
        L, F, G, s = _lib.lib(), self.F, self.G, stream.cuda_stream
        nt = self.n_tri.data_ptr()
        _lib.check(L.opcfe_narrow_indices(self.trimap.data_ptr(), self.trimap32.data_ptr(), F,
                                          G, 1, None, G, G, s), "narrow_indices")
        _lib.check(L.opcfe_narrow_indices(self.triangles.data_ptr(), self.triangles32.data_ptr(),
                                          F, G, 3, nt, 3 * G, 3 * G, s), "narrow_indices")
        if self.halfedges32 is not None:
            _lib.check(L.opcfe_narrow_indices(self.halfedges.data_ptr(),
                                              self.halfedges32.data_ptr(), F, G, 3, nt, 3 * G,
                                              3 * G, s), "narrow_indices")

    def _capture(self):
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self._launch(s)                                     # warm-up (lazy attrs, TMA encode)
        torch.cuda.current_stream(self.device).wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            self._launch(s)
        self._graph = g

    def launch(self):
        """Enqueue one batch on the current stream (inputs already in self.src)."""
        if self._use_graph:
            if self._graph is None:
                self._capture()
            self._graph.replay()
        else:
            self._launch(torch.cuda.current_stream(self.device))

    def launch_profiled(self, events):
        """Enqueue one batch without the graph, recording 5 stage-boundary CUDA events
        ([0] start, [1] after stage-in, [2] after Laplacian, [3] after triangulation,
        [4] end) on the current stream -- the reference's per-stage _Timer
        (pipeline.py:55-68) measured on the device."""
        arr = (ctypes.c_void_p * 5)(*[None if e is None else e.cuda_event for e in events])
        s = torch.cuda.current_stream(self.device)
        rc = _lib.lib().opcfe_front_end_profiled(self.F, self.M, self.N, ctypes.byref(self.p),
                                                 ctypes.byref(self.io), self.ws.data_ptr(),
                                                 self.ws.numel(), s.cuda_stream, arr)
        _lib.check(rc, "front_end_profiled")
        self._narrow(s)

    def run(self, src: torch.Tensor | None = None) -> FrontEndResult:
        """Process the batch in self.src (or copy `src` (F,M,N,3) into it first)."""
        if src is not None:
            self.src.copy_(src.reshape(self.src.shape))
        self.launch()
        return self.result()

    def device_outputs(self) -> dict:
        """name -> (device tensor (F, ...), rows-per-triangle: 0 = fixed size) of every
        output this engine produces, index arrays in self.index_dtype."""
        c = self.index_dtype == torch.int32
        out = {"points": (self.points_view(), 0),
               "trimap": (self.trimap32 if c else self.trimap, 0),
               "triangles": (self.triangles32 if c else self.triangles, 1),
               "halfedges": (self.halfedges32 if c else self.halfedges, 3),
               "normals": (self.normals, 1), "lmax": (self.lmax, 1), "labels": (self.labels, 1)}
        return {k: v for k, v in out.items() if v[0] is not None}

    def points_view(self) -> torch.Tensor:
        """The smoothed grid as (F, M, N, 3) (fast: a view of the padded fp32 rows)."""
        if self.f64:
            return self.grid
        return self.grid[..., :3 * self.N].unflatten(-1, (self.N, 3))

    def result(self) -> FrontEndResult:
        pts = self.points_view()
        return FrontEndResult(points=pts, triangles=self.triangles, trimap=self.trimap,
                              halfedges=self.halfedges, normals=self.normals,
                              lmax_mask=self.lmax, n_tri=self.n_tri.tolist(), labels=self.labels,
                              grid_shape=(self.M, self.N))

    # -------------------------------------------------------------------- host
    def host_buffers(self):
        """Pinned host destinations for run_host (allocated once)."""
        if not hasattr(self, "_host"):
            F, M, N, G = self.F, self.M, self.N, self.G
            pin = dict(pin_memory=True)
            fdt = self.grid.dtype
            self._host = dict(
                points=torch.empty((F, M, N, 3), dtype=fdt, **pin),
                trimap=torch.empty((F, G), dtype=torch.int64, **pin),
                triangles=torch.empty((F, G, 3), dtype=torch.int64, **pin),
                halfedges=torch.empty((F, 3 * G), dtype=torch.int64, **pin) if self.halfedges is not None else None,
                normals=torch.empty((F, G, 3), dtype=fdt, **pin) if self.normals is not None else None,
                lmax=torch.empty((F, G), dtype=torch.uint8, **pin) if self.lmax is not None else None,
                n_tri=torch.empty((F,), dtype=torch.int64, **pin),
            )
        return self._host

    def run_host(self, src_host: torch.Tensor) -> FrontEndResult:
        """End to end through host memory: H2D(src) -> front end -> D2H(all outputs).

        `src_host` is a pinned (F,M,N,3) tensor of self.src's dtype.  Outputs land
        in pinned host buffers (see host_buffers); returns them as a FrontEndResult.
        Returns the number of bytes moved as attributes h2d_bytes / d2h_bytes.
        """
        H = self.host_buffers()
        cur = torch.cuda.current_stream(self.device)
        self.src.copy_(src_host, non_blocking=True)
        self.launch()
        H["n_tri"].copy_(self.n_tri, non_blocking=True)
        cur.synchronize()                                        # data-dependent sizes
        nt = H["n_tri"].tolist()
        d2h = 8 * self.F
        H["points"].copy_(self.points_view(), non_blocking=True)
        H["trimap"].copy_(self.trimap, non_blocking=True)
        fsz = self.grid.element_size()
        d2h += H["points"].numel() * fsz + H["trimap"].numel() * 8
        for f, T in enumerate(nt):
            H["triangles"][f, :T].copy_(self.triangles[f, :T], non_blocking=True)
            d2h += 24 * T
            if H["halfedges"] is not None:
                H["halfedges"][f, :3 * T].copy_(self.halfedges[f, :3 * T], non_blocking=True)
                d2h += 24 * T
            if H["normals"] is not None:
                H["normals"][f, :T].copy_(self.normals[f, :T], non_blocking=True)
                d2h += 3 * fsz * T
            if H["lmax"] is not None:
                H["lmax"][f, :T].copy_(self.lmax[f, :T], non_blocking=True)
                d2h += T
        cur.synchronize()
        self.h2d_bytes = src_host.numel() * src_host.element_size()
        self.d2h_bytes = d2h
        return FrontEndResult(points=H["points"], triangles=H["triangles"], trimap=H["trimap"],
                              halfedges=H["halfedges"], normals=H["normals"], lmax_mask=H["lmax"],
                              n_tri=nt, grid_shape=(self.M, self.N))


class HostPipeline:
    """End-to-end frames through host memory with copies overlapped across frames.

    Two FrontEnd slots (each a CUDA graph over `frames_per_slot` frames) and three
    streams: chunk i+1's H2D and front end run while chunk i's outputs stream back (D2H).
    A frame's D2H is sized by its own triangle count (one event wait per chunk on the
    host), so only live rows travel.  Small frames go several to a slot (default: ~32 MB
    of input per slot, at most 64 frames; OPCFE_SLOT_MB / OPCFE_SLOT_MAX), so the per-chunk host wait and launch latency are amortised.

    outputs      which results come back (default: the drop-in set mesh_from_opc +
                 bilateral_filter_opc return -- smoothed grid, trimap, triangles,
                 halfedges, normals; also "lmax" (needs l_max) and "labels" (needs
                 dominant_normals)).  Unrequested outputs are not copied.
    index_dtype  torch.int64 (the reference's dtype) or torch.int32 -- compact,
                 NON-reference indices narrowed on the device (half the index bytes).
    precision    "fast" (fp32 outputs), "strict" (float64, the reference's chain) or
                 "mixed" (float64; strict up to the FC data, fp32 bilateral).
    """

    DROPIN = ("points", "trimap", "triangles", "halfedges", "normals")
    NAMES = DROPIN + ("lmax", "labels")

    def __init__(self, M, N, laplacian=LaplacianParams(), bilateral=BilateralParams(),
                 l_max=None, src_dtype=torch.float64, device=None, frames_per_slot=None,
                 precision: str = "fast", outputs=DROPIN, index_dtype=torch.int64,
                 dominant_normals=None, ang_min: float = 0.95):
        outputs = tuple(outputs)
        bad = [o for o in outputs if o not in self.NAMES]
        if bad:
            raise ValueError(f"unknown outputs {bad}; choose from {self.NAMES}")
        if "lmax" in outputs and l_max is None:
            raise ValueError("the lmax output needs l_max")
        if "labels" in outputs and dominant_normals is None:
            raise ValueError("the labels output needs dominant_normals")
        if frames_per_slot is None:
            esz = torch.empty((), dtype=src_dtype).element_size()
            frames_per_slot = max(1, min(int(os.environ.get("OPCFE_SLOT_MAX", "64")),
                                         (int(os.environ.get("OPCFE_SLOT_MB", "32")) << 20)
                                         // (M * N * 3 * esz)))
        self.k = k = int(frames_per_slot)
        self.outputs = outputs
        self.slots = [FrontEnd(M, N, k, laplacian=laplacian, bilateral=bilateral, l_max=l_max,
                               halfedges="halfedges" in outputs,
                               normals="normals" in outputs or "labels" in outputs,
                               dominant_normals=dominant_normals, ang_min=ang_min,
                               src_dtype=src_dtype, device=device, graph=True,
                               precision=precision, index_dtype=index_dtype)
                      for _ in range(2)]
        dev = self.slots[0].device
        self.device = dev
        self.M, self.N, self.G = M, N, self.slots[0].G
        self.s_h2d = torch.cuda.Stream(device=dev)
        self.s_cmp = torch.cuda.Stream(device=dev)
        self.s_d2h = torch.cuda.Stream(device=dev)
        self.ev_h2d = [torch.cuda.Event() for _ in range(2)]
        self.ev_cmp = [torch.cuda.Event() for _ in range(2)]
        self.ev_d2h = [torch.cuda.Event() for _ in range(2)]
        self.ntri_host = torch.empty((2, k), dtype=torch.int64, pin_memory=True)
        self._host = None
        self.kernel_launches = self.slots[0].kernel_launches
        for s in self.slots:   # capture both graphs up front
            s.launch()
        torch.cuda.synchronize(dev)

    def host_outputs(self, F):
        if self._host is None or self._host["points"].shape[0] < F:
            # only the requested outputs (points is always sized for the batch bookkeeping)
            dev_out = self.slots[0].device_outputs()
            self._host = {}
            for name in set(self.outputs) | {"points"}:
                t = dev_out[name][0]
                self._host[name] = torch.empty((F,) + tuple(t.shape[1:]), dtype=t.dtype,
                                                pin_memory=True)
        return self._host

    def _enqueue(self, src_host, c):
        s = c % 2
        eng = self.slots[s]
        lo = c * self.k
        n = min(self.k, src_host.shape[0] - lo)
        with torch.cuda.stream(self.s_h2d):
            self.s_h2d.wait_event(self.ev_cmp[s])      # slot input consumed by chunk c-2
            eng.src[:n].copy_(src_host[lo:lo + n], non_blocking=True)
            self.ev_h2d[s].record(self.s_h2d)
        with torch.cuda.stream(self.s_cmp):
            self.s_cmp.wait_event(self.ev_h2d[s])
            self.s_cmp.wait_event(self.ev_d2h[s])      # slot outputs drained (chunk c-2)
            eng._graph.replay()
            self.ntri_host[s].copy_(eng.n_tri, non_blocking=True)
            self.ev_cmp[s].record(self.s_cmp)

    def _drain(self, H, c, F):
        s = c % 2
        eng = self.slots[s]
        lo = c * self.k
        n = min(self.k, F - lo)
        self.ev_cmp[s].synchronize()                    # the chunk's n_tri are on the host
        nt = [int(t) for t in self.ntri_host[s, :n]]
        dev_out = eng.device_outputs()
        b = 8 * n
        with torch.cuda.stream(self.s_d2h):
            self.s_d2h.wait_event(self.ev_cmp[s])
            for name in self.outputs:
                t, per_tri = dev_out[name]
                if per_tri == 0:                        # fixed-size per frame
                    H[name][lo:lo + n].copy_(t[:n], non_blocking=True)
                    b += t[:n].numel() * t.element_size()
                    continue
                for j, T in enumerate(nt):
                    rows = per_tri * T
                    H[name][lo + j, :rows].copy_(t[j, :rows], non_blocking=True)
                    b += t[j, :rows].numel() * t.element_size()
            self.ev_d2h[s].record(self.s_d2h)
        return nt, b

    def run(self, src_host: torch.Tensor) -> FrontEndResult:
        """src_host: pinned (F, M, N, 3).  Returns pinned host outputs (valid until the
        next run); every copy has completed when run() returns."""
        F = src_host.shape[0]
        H = self.host_outputs(F)
        for s in (self.s_h2d, self.s_cmp, self.s_d2h):
            s.wait_stream(torch.cuda.current_stream(self.device))
        chunks = (F + self.k - 1) // self.k
        nt, d2h = [], 0
        self._enqueue(src_host, 0)
        for c in range(chunks):
            if c + 1 < chunks:
                self._enqueue(src_host, c + 1)
            t, b = self._drain(H, c, F)
            nt += t
            d2h += b
        torch.cuda.current_stream(self.device).wait_stream(self.s_d2h)
        self.s_d2h.synchronize()                        # host buffers complete
        self.h2d_bytes = src_host.numel() * src_host.element_size()
        self.d2h_bytes = d2h
        get = lambda k: H[k][:F] if k in self.outputs else None
        return FrontEndResult(points=get("points"), triangles=get("triangles"),
                              trimap=get("trimap"), halfedges=get("halfedges"),
                              normals=get("normals"), lmax_mask=get("lmax"), n_tri=nt,
                              grid_shape=(self.M, self.N), labels=get("labels"))


_ENGINES_MAX = 4
_ENGINES_TLS = threading.local()


def cached_engine(M, N, laplacian, bilateral, l_max, src_dtype, precision, frames=1,
                  dominant_normals=None, ang_min=0.95, device=None) -> FrontEnd:
    """A FrontEnd for these shapes / parameters, reused across calls (buffers, workspace
    and TMA descriptors are built once; a small LRU per THREAD, so concurrent callers
    never share an engine's buffers -- the reference's functions are reentrant)."""
    from collections import OrderedDict
    _ENGINES = getattr(_ENGINES_TLS, "engines", None)
    if _ENGINES is None:
        _ENGINES = _ENGINES_TLS.engines = OrderedDict()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    dn_key = None if dominant_normals is None else \
        np.asarray(dominant_normals, dtype=np.float64).tobytes()
    key = (M, N, frames, laplacian and (laplacian.lam, laplacian.kernel_size, laplacian.iterations),
           bilateral and (bilateral.sigma_length, bilateral.sigma_angle, bilateral.kernel_size,
                          bilateral.iterations),
           l_max, src_dtype, precision, dn_key, ang_min, dev)
    eng = _ENGINES.get(key)
    if eng is None:
        eng = FrontEnd(M, N, frames, laplacian=laplacian, bilateral=bilateral, l_max=l_max,
                       dominant_normals=dominant_normals, ang_min=ang_min, src_dtype=src_dtype,
                       device=dev, graph=False, precision=precision)
        _ENGINES[key] = eng
        while len(_ENGINES) > _ENGINES_MAX:
            _ENGINES.popitem(last=False)
    else:
        _ENGINES.move_to_end(key)
    return eng


def front_end(opc, laplacian: LaplacianParams | None = None,
              bilateral: BilateralParams | None = None, l_max: float | None = None,
              precision: str | None = None):
    """Single-frame organized front-end (pipeline.py:125-134) on the GPU.

    Returns (smoothed grid, HalfEdgeMesh, l_max mask or None); NumPy in ->
    NumPy out (float arrays as float64 like the reference), torch in -> torch.
    Precision as smoothing.resolve_precision (float64 input: the reference's fp64
    chain by default).  Engines are cached per shape and parameters.
    """
    from .smoothing import resolve_precision
    is_np = not isinstance(opc, torch.Tensor)
    src = host_view(np.ascontiguousarray(opc, dtype=np.float64)) if is_np else opc
    if src.dtype not in (torch.float32, torch.float64):
        src = src.to(torch.float64)
    src = src.to("cuda").contiguous()
    M, N = src.shape[:2]
    prec = resolve_precision(precision, src.dtype)
    eng = cached_engine(M, N, laplacian, bilateral, l_max, src.dtype, prec)
    res = eng.run(src.unsqueeze(0))
    mesh = res.mesh(0)
    if is_np:
        conv = lambda t, dt=None: None if t is None else (t.cpu().numpy() if dt is None
                                                          else t.cpu().numpy().astype(dt))
        smoothed = conv(res.points[0], np.float64)
        mesh = HalfEdgeMesh(points=smoothed.reshape(-1, 3), triangles=conv(mesh.triangles),
                            halfedges=conv(mesh.halfedges), normals=conv(mesh.normals, np.float64),
                            trimap=conv(mesh.trimap), grid_shape=(M, N))
        mask = None if res.lmax_mask is None else conv(res.lmax_mask[0, :mesh.num_triangles]).astype(bool)
        return smoothed, mesh, mask
    # torch callers: copies, so the next call on the cached engine cannot alias them
    cl = lambda t: None if t is None else t.clone()
    pts = res.points[0].clone()
    mesh = HalfEdgeMesh(points=pts.reshape(-1, 3), triangles=cl(mesh.triangles),
                        halfedges=cl(mesh.halfedges), normals=cl(mesh.normals),
                        trimap=cl(mesh.trimap), grid_shape=(M, N))
    mask = None if res.lmax_mask is None else res.lmax_mask[0, :len(mesh.triangles)].bool()
    return pts, mesh, mask
