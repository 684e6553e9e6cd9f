#!/usr/bin/env python
"""Benchmark: frames/s of the organized front-end (Laplacian + mesh + bilateral) on 1080p.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

Workload (BASELINE.json configs[3], the config the metric is quoted on): 1080x1920
organized clouds, 10 Laplacian (lam 1, k 3) + 5 bilateral (sl 0.1, sa 0.15, k 3)
iterations, full mesh + half-edge twins.  A step = one batch of F frames per GPU
(F * 25 MB fp32 input > L2, so every step streams from HBM).  Frames are
independent: ranks shard batches, no collective on the data path (weak scaling).

One JSON line on rank 0:
  value      device-resident whole-job frames/s (inputs in HBM, CUDA events, max over ranks)
  e2e        same metric through the host API: pinned f64 host frames -> H2D -> front end
             -> D2H of every mesh output (points, triangles, twins, trimap, normals)
  roofline   dominant kernel: algorithmic bytes / CUDA-event time vs the
             measured HBM copy bandwidth (MEASURED_PEAKS.json)
  cpu_baseline  the reference's own CPU path (oracle/_ref = its compiled Cython kernels)
             on this host's cores, on a bounded sample
--impl reference times only that CPU path (rank 0) and prints the same line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "frames/sec (HBM GB/s vs roofline) for smooth+mesh of 1080p organized PC, 1/2/4/8 GPU"


class Workload:
    """One of BASELINE.json's configs.  C4 (the metric's config) is the default bench
    line; the others are secondary lines (`--workload`), C5 strong-scales a fixed batch."""

    def __init__(self, name, desc, M, N, lap, bil, l_max, base, frames, total=None,
                 dropout=0.0):
        self.name, self.desc, self.M, self.N = name, desc, M, N
        self.lap, self.bil, self.l_max, self.base = lap, bil, l_max, base
        self.frames, self.total, self.dropout = frames, total, dropout


def _base(name):
    def make():
        from paper_2007_12065_b200 import synthetic
        return getattr(synthetic, name)()
    return make


WORKLOADS = {
    "C4": Workload("C4", "C4: 1080x1920 organized cloud (room scene), 10 Laplacian + 5 bilateral "
                         "iterations, full mesh + half-edge twins",
                   1080, 1920, (1.0, 3, 10), (0.1, 0.15, 3, 5), None, _base("config_c4"), 16),
    "C1": Workload("C1", "C1: 250x250 room scene, 1 Laplacian + 1 bilateral iteration",
                   250, 250, (1.0, 3, 1), (0.1, 0.15, 3, 1), None, _base("config_c1"), 256),
    "C2": Workload("C2", "C2: 480x640 RealSense-sized room crop (2 % dropout), 3 Laplacian + 2 "
                         "bilateral iterations, mesh + normals",
                   480, 640, (1.0, 3, 3), (0.1, 0.15, 3, 2), None, _base("config_c2"), 64),
    "C3": Workload("C3", "C3: 64x1024 LiDAR range image with NaN gaps, 5 Laplacian iterations, "
                         "l_max = 0.5 mask, mesh + twins + normals",
                   64, 1024, (1.0, 3, 5), None, 0.5, _base("config_c3"), 512),
    "C5": Workload("C5", "C5: batch of 512 frames at 480x640 (C2 base + per-frame 2 mm noise + "
                         "2 % dropout) split over the GPUs, full front-end per frame",
                   480, 640, (1.0, 3, 3), (0.1, 0.15, 3, 2), None, _base("config_c5_base"),
                   512, total=512, dropout=0.02),
}
WL = WORKLOADS["C4"]


def config_dict(frames, wl=None):
    wl = wl or WL
    per = frames * wl.M * wl.N * 12
    return {"workload": wl.desc,
            "frames_per_gpu_per_step": frames, "grid": [wl.M, wl.N],
            "laplacian": ({"lam": wl.lap[0], "kernel_size": wl.lap[1], "iterations": wl.lap[2]}
                          if wl.lap else None),
            "bilateral": ({"sigma_length": wl.bil[0], "sigma_angle": wl.bil[1],
                           "kernel_size": wl.bil[2], "iterations": wl.bil[3]} if wl.bil else None),
            **({"l_max": wl.l_max} if wl.l_max is not None else {}),
            **({"total_frames_per_step": wl.total} if wl.total else {}),
            "l2": (f"inputs larger than L2: {frames} x {wl.M * wl.N * 12 / 1e6:.1f} MB fp32 "
                   f"= {per / 1e6:.0f} MB per step per GPU" if per > 126e6 else
                   f"inputs {per / 1e6:.0f} MB per step per GPU: L2-resident (126 MB L2), "
                   "flagged per SURVEY.md 8d"),
            "outputs": "smoothed grid fp32, triangles/trimap/halfedges int64, normals fp32"
                       + (", l_max flags u8" if wl.l_max is not None else "")}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.start = self.stop = 0

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()                    # nvidia-smi takes ~0.1-0.3 s to start:
            while not self.rows and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)                # sample only once it is streaming
        except OSError:
            self.proc = None
        self.start = len(self.rows)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        self.stop = len(self.rows)
        if self.proc is not None:
            if self.stop == self.start:         # region shorter than one interval: take
                t0 = time.time()                # the sample that closes it
                while len(self.rows) == self.stop and time.time() - t0 < 0.2:
                    time.sleep(0.005)
                self.stop = len(self.rows)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        load = [r for r in self.rows[self.start:self.stop]
                if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        if not load:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        mhz = [float(r[0]) for r in load]
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in load:
            for name, v in zip(names, r[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(mhz), "sm_max_mhz": float(load[0][1]),
                "reasons": sorted(reasons), "samples": len(load),
                "power_w_max": max(float(r[2]) for r in load if r[2].replace(".", "").isdigit())}


# ------------------------------------------------------------------ reference arm
def cpu_reference(steps, warmup, budget_s=None, wl=None, want_sample=False):
    """Time the reference's own CPU implementation on this host: one whole frame per
    process per step (small frames: several per task so a step is >= ~0.5 s), stopping
    early once `budget_s` of timed work is done.  With want_sample, worker 0's outputs
    of the first timed step are returned for the chained-parity check."""
    import numpy as np
    from oracle import ref_frontend
    wl = wl or WL
    frame = wl.base()
    cores = len(os.sched_getaffinity(0))
    per_task = max(1, int(round(0.5 / _ref_frame_seconds(wl))))
    pool = ref_frontend.ReferencePool(frame, cores, wl.lap, wl.bil, frames_per_task=per_task)
    sample = None
    try:
        for _ in range(warmup):
            pool.step()
        times, credit = [], 0
        for k in range(steps):
            dt, fr, smp = pool.step(want_sample=want_sample and k == 0)
            sample = sample or smp
            times.append(dt)
            credit += fr
            if budget_s is not None and sum(times) > budget_s:
                break
    finally:
        pool.close()
    total = sum(times)
    return {"value": credit / total, "unit": "frames/s", "cores": cores,
            "kind": ref_frontend.kind(),
            "sample": f"{len(times)} timed steps (+{warmup} warm-up) x {cores} processes, each "
                      f"{per_task} whole {wl.M}x{wl.N} {wl.name} frame(s) per step through "
                      f"{ref_frontend.path_name()}; single-threaded math per process; "
                      f"CPU: {ref_frontend.cpu_model()}",
            "cpu_model": ref_frontend.cpu_model(),
            "ms_per_step": 1e3 * total / len(times), "steps_timed": len(times),
            "frames_per_step": cores * per_task, "np_version": np.__version__}, sample


def _ref_frame_seconds(wl):
    """Rough single-core seconds per frame of the reference, used
    only to size a step; C4 ~12 s, scaling with points and iterations."""
    P = wl.M * wl.N
    lap = wl.lap[2] if wl.lap else 0
    bil = wl.bil[3] if wl.bil else 0
    return P * (0.075e-6 * lap + 0.86e-6 * bil + 1.5e-6)


def run_reference(args, rank, world, wl):
    if rank != 0:
        return 0
    # whole frames cost ~12 s of CPU each at C4: warm-up capped at 1 step, timed steps
    # stop after ~150 s so the default --steps 200 run ends within a few minutes
    cb, _ = cpu_reference(args.steps, min(args.warmup, 1), budget_s=150.0, wl=wl)
    line = {"metric": METRIC, "value": cb["value"], "unit": "frames/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": cb["steps_timed"], "warmup": min(args.warmup, 1),
            "ms_per_step": cb["ms_per_step"], "higher_is_better": True,
            "scaling": "strong" if wl.total else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args.frames, wl),
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "steps_note": f"--steps {args.steps} requested; whole-frame steps stop after 150 s "
                          "of timed work (steps = the steps actually timed)"}
    print(json.dumps(line), flush=True)
    return 0


def chained_parity(sample, wl, dev):
    """GPU chain vs the reference's OWN chain on the same whole frame (worker 0's output of
    the cpu_baseline leg): fast (fp32), mixed and strict (fp64) precision."""
    import numpy as np
    import torch

    import paper_2007_12065_b200 as fe
    base = wl.base()
    M, N = base.shape[:2]
    ref_sm, ref_n, ref_tm = sample["smoothed"], sample["normals"], sample["trimap"]
    ok = np.isfinite(ref_sm).all(2)
    out = {"frame": f"{wl.name} base frame {M}x{N} (the cpu_baseline leg's worker 0)"}
    for prec in ("fast", "mixed", "strict"):
        eng = fe.FrontEnd(M, N, 1, laplacian=fe.LaplacianParams(*wl.lap) if wl.lap else None,
                          bilateral=fe.BilateralParams(*wl.bil) if wl.bil else None,
                          l_max=wl.l_max, src_dtype=torch.float64, device=dev, graph=False,
                          precision=prec)
        res = eng.run(torch.from_numpy(base).to(dev).unsqueeze(0))
        torch.cuda.synchronize(dev)
        T = res.n_tri[0]
        sm = res.points[0].cpu().numpy().astype(np.float64)
        tm = res.trimap[0].cpu().numpy()
        he_linked = int((res.halfedges[0, :3 * T] >= 0).sum().item())
        g_n = res.normals[0, :T].cpu().numpy().astype(np.float64)
        verr = np.linalg.norm(sm[ok] - ref_sm[ok], axis=1) / \
            np.maximum(np.linalg.norm(ref_sm[ok], axis=1), 1e-300)
        nok = ~np.isnan(ref_n).any(1)
        nerr = np.linalg.norm(g_n[nok] - ref_n[nok], axis=1) if T == len(ref_n) else None
        q = lambda e: None if e is None or e.size == 0 else float(np.quantile(e, 0.999))
        out[prec] = {
            "topology_exact": bool(np.array_equal(tm, ref_tm) and
                                   he_linked == sample["n_halfedges_linked"]),
            "smoothed_bit_exact": bool(np.array_equal(np.nan_to_num(sm), np.nan_to_num(ref_sm))
                                       and np.array_equal(np.isnan(sm), np.isnan(ref_sm))),
            "smoothed_rel": {"max": float(verr.max()) if verr.size else 0.0, "p99.9": q(verr),
                             "n_over_1e-5": int((verr > 1e-5).sum()), "n": int(verr.size)},
            "normals_abs": None if nerr is None else {
                "max": float(nerr.max()) if nerr.size else 0.0, "p99.9": q(nerr),
                "n_over_1e-5": int((nerr > 1e-5).sum()), "n": int(nerr.size)},
        }
        del eng, res
        torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------ our arm
def algorithmic_bytes(frames, T, wl=None):
    """SURVEY.md 8d per-frame algorithmic bytes (fp32 AoS, int64 indices, per pass)."""
    wl = wl or WL
    P = wl.M * wl.N
    Q = (wl.M - 1) * (wl.N - 1)
    G = 2 * Q
    lap_it = wl.lap[2] if wl.lap else 0
    bil_it = wl.bil[3] if wl.bil else 0
    # triangulation: points in, trimap (+ its read-back for twins), triangles + twins out;
    # + the l_max flags (T bytes); without bilateral the mesh-order normals (12T) too
    tri = 12 * P + 16 * G + 48 * T + (T if wl.l_max is not None else 0) + (0 if wl.bil else 12 * T)
    # bilateral stage: FC normals+centroids (12P + 48Q) + 72Q per iteration +
    # mesh-order gather (12G + 12T); per launch = stage / iterations
    bil = ((12 * P + 48 * Q) + bil_it * 72 * Q + 12 * G + 12 * T) if wl.bil else 0
    return {
        "laplacian_per_launch": frames * 24 * P,
        "triangulate_per_launch": frames * tri,
        "bilateral_stage": frames * bil,
        "frame_total": 24 * P * lap_it + tri + bil,
    }


def load_peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_fp32_peak():
    p = os.path.join(REPO, "profiles", "fp32_peak.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)["fp32_lane_ops_per_s"], "measured (profiles/fp32_peak.json)"
    return 148 * 128 * 1.965e9, "nominal 128 FP32 lanes/clk/SM at 1965 MHz"


def load_traffic():
    p = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


PRECISION_WHAT = {
    "strict": "precision='strict': the reference's fp64 chain (bit-exact Laplacian, FC data "
              "and topology; bilateral normals within a few ulp per iteration), float64 outputs",
    "mixed": "precision='mixed': a float64 Laplacian with rsqrt pair weights (vertices "
             "within a few ulp), exact topology and FC data, then the fp32 bilateral on the "
             "FC arrays -- normals within 1e-5 of the reference's chain end to end "
             "(parity.chained.mixed), float64 outputs",
}


def precision_throughput(fe, wl, eng_fast, args, dev, precision="strict"):
    """Device-resident frames/s of the STRICT (the reference's fp64 arithmetic) or MIXED
    chain on the same frames as the fast line (eng_fast.src), CUDA events on the launching
    stream."""
    import torch
    F = eng_fast.F
    eng = fe.FrontEnd(wl.M, wl.N, F, laplacian=fe.LaplacianParams(*wl.lap) if wl.lap else None,
                      bilateral=fe.BilateralParams(*wl.bil) if wl.bil else None, l_max=wl.l_max,
                      src_dtype=eng_fast.src.dtype, device=dev, graph=False, precision=precision)
    eng.src.copy_(eng_fast.src)
    stream = torch.cuda.current_stream(dev)
    for _ in range(2):
        eng.launch()
    steps = 5
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    a.record(stream)
    for _ in range(steps):
        eng.launch()
    b.record(stream)
    torch.cuda.synchronize(dev)
    ms = a.elapsed_time(b) / steps
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    for e in ev:                                    # materialise the cudaEvent_t handles
        e.record(stream)
    eng.launch_profiled(ev)
    torch.cuda.synchronize(dev)
    stage = {"stage_in": ev[0].elapsed_time(ev[1]), "laplacian": ev[1].elapsed_time(ev[2]),
             "triangulate": ev[2].elapsed_time(ev[3]), "bilateral": ev[3].elapsed_time(ev[4])}
    out = {"value": F / (ms / 1e3), "unit": "frames/s", "ms_per_step": ms, "frames_per_step": F,
           "steps": steps, "dtype": "f64", "gpu_launches_per_step": eng.kernel_launches,
           "stage_ms_per_step": {k: round(v, 4) for k, v in stage.items()},
           "what": PRECISION_WHAT[precision]}
    del eng
    torch.cuda.empty_cache()
    return out


def dropin_e2e(fe, wl, frame, dev, frames=5):
    """pipeline.py:125-134 unchanged, through the drop-in API (NumPy float64 in, NumPy
    out, one frame per call), host wall clock around each whole frame."""
    import numpy as np
    import torch
    frame = np.ascontiguousarray(frame, dtype=np.float64)
    lp = fe.LaplacianParams(*wl.lap) if wl.lap else None
    bp = fe.BilateralParams(*wl.bil) if wl.bil else None

    def one():
        sm = fe.laplacian_filter_opc(frame, lp) if lp else frame
        mesh = fe.mesh_from_opc(sm)
        if bp:
            mesh.normals = fe.bilateral_filter_opc(sm, bp, mesh.trimap)
        return sm, mesh

    # warm-up as the timed loop runs (the previous frame's results alive while the next
    # is computed), so the pinned result blocks of both are cached before timing
    sm, mesh = one()
    sm, mesh = one()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(frames):
        sm, mesh = one()
    dt = (time.perf_counter() - t0) / frames
    T = mesh.num_triangles
    h2d = 3 * frame.nbytes + mesh.trimap.nbytes     # opc to each call + the trimap
    d2h = sm.nbytes + mesh.triangles.nbytes + mesh.halfedges.nbytes + mesh.trimap.nbytes + \
        24 * T * (2 if bp else 1)
    from paper_2007_12065_b200 import smoothing
    return {"value": 1.0 / dt, "unit": "frames/s", "frames": frames,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "precision": smoothing.resolve_precision(None, torch.float64),
            "path": "laplacian_filter_opc -> mesh_from_opc -> bilateral_filter_opc on NumPy "
                    "float64 (pageable) arrays, one frame per call, host wall clock"}


PLUGIN_CHILD = r"""
import json, sys, time
import numpy as np
from flatpoly import _kernels, mesh, smoothing
assert _kernels.ACTIVE == "cuda", _kernels.ACTIVE
opc = np.load(sys.argv[1])
cfg = json.loads(sys.argv[2])
lp = smoothing.LaplacianParams(*cfg["lap"]) if cfg["lap"] else None
bp = smoothing.BilateralParams(*cfg["bil"]) if cfg["bil"] else None
def one():
    sm = smoothing.laplacian_filter_opc(opc, lp) if lp else opc
    m = mesh.mesh_from_opc(sm)
    if bp:
        m.normals = smoothing.bilateral_filter_opc(sm, bp, m.trimap)
    return sm, m
sm, m = one()
sm, m = one()
n = cfg["frames"]
t = time.perf_counter()
for _ in range(n):
    sm, m = one()
dt = (time.perf_counter() - t) / n
print(json.dumps({"dt": dt, "T": int(m.num_triangles), "sm": int(sm.nbytes),
                  "tm": int(m.trimap.nbytes)}))
"""


def plugin_e2e(wl, frame, frames=5):
    """pipeline.py:125-134 run by the STOCK reference package with libopcfe plugged into
    its own kernel switch (integration/: FLATPOLY_CUDA=1 -- the maintainer's binding over
    the C ABI, strict precision), NumPy f64 in and out, one frame per call, host wall
    clock.  Needs the reference install in baseline/_ref."""
    import subprocess
    import tempfile
    import numpy as np
    ref = os.path.join(REPO, "baseline", "_ref", "flatpoly")
    if not os.path.isdir(ref):
        return {"unavailable": "baseline/_ref missing (baseline/install_ref.sh)"}
    with tempfile.TemporaryDirectory(prefix="flatpoly_cuda_") as dest:
        subprocess.run([sys.executable, os.path.join(REPO, "integration", "install.py"), dest],
                       check=True, stdout=subprocess.DEVNULL)
        fpath = os.path.join(dest, "frame.npy")
        np.save(fpath, np.ascontiguousarray(frame, dtype=np.float64))
        cfg = {"lap": list(wl.lap) if wl.lap else None, "bil": list(wl.bil) if wl.bil else None,
               "frames": frames}
        env = dict(os.environ, FLATPOLY_CUDA="1",
                   OPCFE_LIB=os.path.join(REPO, "paper_2007_12065_b200", "lib", "libopcfe.so"),
                   PYTHONPATH=os.pathsep.join([dest, os.path.join(REPO, "tests", "golden",
                                                                  "_stubs")]))
        r = subprocess.run([sys.executable, "-c", PLUGIN_CHILD, fpath, json.dumps(cfg)], env=env,
                           cwd=dest, capture_output=True, text=True, timeout=600)
    if r.returncode != 0:
        return {"unavailable": "plugin run failed: " + r.stderr.strip().splitlines()[-1][:200]}
    o = json.loads(r.stdout.strip().splitlines()[-1])
    T, fb = o["T"], frame.size * 8
    # uploads: the cloud to the Laplacian, the smoothed cloud to mesh_from_opc and (+ the
    # trimap) to bilateral_filter_opc; downloads: the smoothed cloud, triangles, trimap,
    # twins and normals of the mesh, the filtered normals
    h2d = (fb if wl.lap else 0) + fb + ((fb + o["tm"]) if wl.bil else 0)
    d2h = (o["sm"] if wl.lap else 0) + 3 * 24 * T + o["tm"] + (24 * T if wl.bil else 0)
    return {"value": 1.0 / o["dt"], "unit": "frames/s", "frames": frames,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "path": "the stock reference package (baseline/_ref) with the shipped binding "
                    "(integration/_opcfe.py + flatpoly_cuda.patch, FLATPOLY_CUDA=1): its own "
                    "laplacian_filter_opc -> mesh_from_opc -> bilateral_filter_opc calling "
                    "libopcfe through ctypes, strict precision, NumPy float64 in and out, one "
                    "frame per call, host wall clock"}


def gpu_index(local_rank, args):
    """The rank's CUDA device: LOCAL_RANK, or LOCAL_RANK % device_count under --share-gpus."""
    import torch
    n = torch.cuda.device_count()
    if args.share_gpus:
        return local_rank % max(n, 1)
    if local_rank >= n:
        raise SystemExit(f"LOCAL_RANK {local_rank} but only {n} CUDA device(s); "
                         "use --share-gpus for a dry run")
    return local_rank


def run_ours(args, rank, world, local_rank, wl):
    import torch
    import torch.distributed as dist

    import paper_2007_12065_b200 as fe
    from paper_2007_12065_b200 import distributed as D

    gpu = gpu_index(local_rank, args)
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    M, N = wl.M, wl.N
    lap_p = fe.LaplacianParams(*wl.lap) if wl.lap else None
    bil_p = fe.BilateralParams(*wl.bil) if wl.bil else None
    if wl.total:          # a fixed batch split over the ranks (strong scaling)
        lo, hi = D.shard_range(wl.total, world, rank)
        F = hi - lo
    else:                 # F frames per GPU per step (weak scaling)
        F = args.frames
    base = torch.from_numpy(wl.base()).to(dev, torch.float32)
    g = torch.Generator(device=dev)
    g.manual_seed(1000 + rank)
    frames = base.unsqueeze(0) + 0.002 * torch.randn((F, M, N, 3), generator=g, device=dev)
    if wl.dropout:
        drop = torch.rand((F, M, N, 1), generator=g, device=dev) < wl.dropout
        frames.masked_fill_(drop, float("nan"))
    eng = fe.FrontEnd(M, N, F, laplacian=lap_p, bilateral=bil_p, l_max=wl.l_max,
                      src_dtype=torch.float32, graph=False)
    eng.src.copy_(frames)
    del frames
    stream = torch.cuda.current_stream(dev)
    prof_steps = max(1, min(args.steps, 20))
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(prof_steps)]
    for row in ev:                                  # materialise the cudaEvent_t handles
        for e in row:
            e.record(stream)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # the measured step: opcfe_front_end as a user calls it (Laplacian -> triangulation ->
    # bilateral on the caller's stream)
    for _ in range(args.warmup):
        eng.launch()
    barrier()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(gpu) as clk:
        barrier()
        t_start.record(stream)
        for k in range(args.steps):
            eng.launch()
        t_end.record(stream)
        barrier()
    elapsed_ms = t_start.elapsed_time(t_end)
    # per-stage device times: opcfe_front_end_profiled runs the stages back to back with
    # stage-boundary events (the reference's _Timer stages), on separate steps
    for _ in range(2):
        eng.launch_profiled(ev[0])
    for k in range(prof_steps):
        eng.launch_profiled(ev[k])
    torch.cuda.synchronize()
    stage = {"stage_in": [], "laplacian": [], "triangulate": [], "bilateral": []}
    for row in ev:
        stage["stage_in"].append(row[0].elapsed_time(row[1]))
        stage["laplacian"].append(row[1].elapsed_time(row[2]))
        stage["triangulate"].append(row[2].elapsed_time(row[3]))
        stage["bilateral"].append(row[3].elapsed_time(row[4]))
    stage_ms = {k: sum(v) / len(v) for k, v in stage.items()}
    T = int(eng.n_tri[0].item())
    # max over ranks (device time)
    max_ms = D.max_over_ranks(elapsed_ms, dev)
    dist_info = None
    if world > 1:
        dist_info = {"backend": dist.get_backend(), "world": world,
                     "frames_this_rank": F, "frames_all_ranks": int(D.sum_over_ranks(F, dev)),
                     "devices_visible": torch.cuda.device_count(),
                     "shared_gpu": bool(args.share_gpus)}
        if args.share_gpus:
            dist_info["note"] = ("ranks share GPUs (--share-gpus): a plumbing check of the "
                                 "multi-rank path, NOT a scaling measurement")
    value = (wl.total if wl.total else world * F) * args.steps / (max_ms / 1e3)

    # ---------------- e2e through the host API (pinned f64 host frames -> outputs on host)
    e2e = None
    if not args.no_e2e:
        pipe = fe.HostPipeline(M, N, laplacian=lap_p, bilateral=bil_p, l_max=wl.l_max,
                               src_dtype=torch.float64, device=dev)
        # e2e batch: >= 16 frames (OPCFE_E2E_FRAMES) or ~400 MB of f64 input per run(), at
        # most the step's frames (C4: 16 frames, ~5.7 GB of pinned in/out buffers; the
        # pipeline's fill / drain amortises over the batch: 16 vs 8 frames +2-3 %)
        FE = min(F, max(int(os.environ.get("OPCFE_E2E_FRAMES", "16")), int(400e6 // (M * N * 24))))
        host = torch.empty((FE, M, N, 3), dtype=torch.float64, pin_memory=True)
        host.copy_(eng.src[:FE].double().cpu())
        pipe.run(host)                              # warm-up (pinned outputs allocated)
        e2e_steps = max(3, min(args.steps, 10))
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            pipe.run(host)
        e1.record(stream)
        barrier()
        te = D.max_over_ranks(e0.elapsed_time(e1), dev)
        e2e = {"value": world * FE * e2e_steps / (te / 1e3), "unit": "frames/s",
               "h2d_bytes_per_step": int(pipe.h2d_bytes), "d2h_bytes_per_step": int(pipe.d2h_bytes),
               "steps": e2e_steps, "frames_per_step": FE,
               "path": "HostPipeline.run: pinned f64 host frames -> H2D -> opcfe_front_end "
                       "(CUDA graph per frame) -> D2H of smoothed grid, trimap, triangles, "
                       "halfedges, normals into pinned host buffers; frame i+1's H2D + compute "
                       "overlap frame i's D2H on separate streams"}
        # ---- the same, starting from frame FILES (binary PLY with "comment grid M N",
        # written here to local /tmp): paper_2007_12065_b200.io.FrameFileReader loads the
        # next batch into a pinned double buffer while HostPipeline runs the current one
        e2e_files = None
        if not args.no_e2e_files:
            import tempfile
            from paper_2007_12065_b200 import io as fio
            tmp = tempfile.mkdtemp(prefix=f"opcfe_bench_r{rank}_")
            try:
                paths = []
                for f in range(FE):
                    paths.append(os.path.join(tmp, f"frame{f}.ply"))
                    fio.write_ply(paths[-1], host[f].numpy().reshape(-1, 3), binary=True,
                                  grid=(M, N))
                seq = paths * e2e_steps
                reader = fio.FrameFileReader(seq, batch=FE)
                barrier()
                e0.record(stream)
                for batch in reader:
                    pipe.run(batch)
                e1.record(stream)
                barrier()
                tf = D.max_over_ranks(e0.elapsed_time(e1), dev)
                e2e_files = {"value": world * len(seq) / (tf / 1e3), "unit": "frames/s",
                             "file_bytes_per_step": int(FE * M * N * 24), "steps": e2e_steps,
                             "path": "FrameFileReader (native PLY reader, pread into pinned "
                                     "buffers, next batch loaded during this one) -> "
                                     "HostPipeline.run as in e2e; files in the page cache"}
            finally:
                import shutil
                shutil.rmtree(tmp, ignore_errors=True)
        e2e["from_files"] = e2e_files
        del pipe
        # ---- strict precision end to end (the reference's fp64 chain, float64 points and
        # normals back, int64 indices: exactly the reference's outputs), then the compact
        # (NON-reference) output modes: int32 indices narrowed on the device, optionally
        # only a subset of the outputs
        for key, outs, kw in (("strict", fe.HostPipeline.DROPIN, dict(precision="strict")),
                              ("mixed", fe.HostPipeline.DROPIN, dict(precision="mixed")),
                              ("compact", fe.HostPipeline.DROPIN, dict(index_dtype=torch.int32)),
                              ("selected", ("points", "triangles", "normals"),
                               dict(index_dtype=torch.int32))):
            if key in ("strict", "mixed") and args.no_strict:
                continue
            p2 = fe.HostPipeline(M, N, laplacian=lap_p, bilateral=bil_p, l_max=wl.l_max,
                                 src_dtype=torch.float64, device=dev, outputs=outs, **kw)
            p2.run(host)
            barrier()
            e0.record(stream)
            for _ in range(e2e_steps):
                p2.run(host)
            e1.record(stream)
            barrier()
            tc = D.max_over_ranks(e0.elapsed_time(e1), dev)
            e2e[key] = {"value": world * FE * e2e_steps / (tc / 1e3), "unit": "frames/s",
                        "h2d_bytes_per_step": int(p2.h2d_bytes),
                        "d2h_bytes_per_step": int(p2.d2h_bytes), "outputs": list(outs),
                        "precision": kw.get("precision", "fast"),
                        "index_dtype": ("int64 (reference)" if "index_dtype" not in kw
                                        else "int32 (non-reference)")}
            del p2
        # ---- the unchanged pipeline.py:125-134 sequence through the drop-in API: NumPy f64
        # in and out, one frame per call (default precision: strict for float64 input)
        if not args.no_e2e_dropin:
            e2e["dropin"] = dropin_e2e(fe, wl, host[0].numpy(), dev)
            if world == 1:
                e2e["plugin"] = plugin_e2e(wl, host[0].numpy())

    if rank != 0:
        return 0
    # ---------------- roofline of the dominant kernel
    peak, peak_src = load_peaks()
    ab = algorithmic_bytes(F, T, wl)
    per_kernel = {"triangulate_kernel": (ab["triangulate_per_launch"], stage_ms["triangulate"], 1)}
    if wl.lap:
        per_kernel["laplacian_kernel"] = (ab["laplacian_per_launch"],
                                          stage_ms["laplacian"] / wl.lap[2], wl.lap[2])
    if wl.bil:
        per_kernel["bilateral_kernel"] = (ab["bilateral_stage"] / wl.bil[3],
                                          stage_ms["bilateral"] / wl.bil[3], wl.bil[3])
    share = {k: v[1] * v[2] for k, v in per_kernel.items()}
    dom = max(share, key=share.get)
    bytes_pl, ms_pl, _ = per_kernel[dom]
    achieved = bytes_pl / (ms_pl / 1e3) / 1e9
    # ncu --set full DRAM bytes of this kernel (profiles/traffic.json), captured at the
    # bench's own batch (16 C4 frames); other batch sizes scale the per-frame figure
    tr = load_traffic().get(dom)
    traffic = None if tr is None else round(tr["dram_bytes_per_launch_per_frame"] * F)
    traffic_src = None if tr is None else (
        f"{tr['capture']}: ncu --set full at {tr['frames']} frames"
        + ("" if tr["frames"] == F else f", scaled to {F} frames"))
    kernels = {k: {"bytes_per_launch": b, "ms_per_launch": round(ms, 4),
                   "GBps": round(b / (ms / 1e3) / 1e9, 1),
                   "frac": round(b / (ms / 1e3) / 1e9 / peak, 3), "launches_per_step": n}
               for k, (b, ms, n) in per_kernel.items()}
    # the bilateral is FP32-bound ("near the FP32/MUFU ridge"): its FP32
    # lane-ops (34 directed pairs per quad at k=3, 15 lane-ops each) vs the FMA pipe
    compute = None
    if wl.bil:
        h = wl.bil[2] // 2
        pairs_per_quad = 2 * (2 * (2 * h + 1) ** 2 - 1)
        fp32_ops = F * (M - 1) * (N - 1) * pairs_per_quad * 15
        fp32_peak, fp32_src = load_fp32_peak()
        fp32_ach = fp32_ops / (stage_ms["bilateral"] / wl.bil[3] / 1e3)
        compute = {"kernel": "bilateral_kernel", "pipe": "fp32 (FMA)",
                   "achieved": round(fp32_ach / 1e12, 2), "peak": round(fp32_peak / 1e12, 2),
                   "unit": "T lane-ops/s", "frac": round(fp32_ach / fp32_peak, 4),
                   "ops_per_launch": fp32_ops, "peak_source": fp32_src,
                   "note": f"{pairs_per_quad} directed pairs per quad x 15 FP32 lane-ops "
                           "(6 differences, 6 squared-distance, 3 accumulate) + 1 MUFU ex2"}
    strict = mixed = None
    if not args.no_strict:
        strict = precision_throughput(fe, wl, eng, args, dev, "strict")
        mixed = precision_throughput(fe, wl, eng, args, dev, "mixed")
    cpu = parity = None
    if world == 1 and not args.no_cpu_baseline:
        cb, sample = cpu_reference(steps=1, warmup=0, budget_s=25.0, wl=wl, want_sample=True)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        if sample is not None:
            parity = {"chained": chained_parity(sample, wl, dev)}
    launches = eng.kernel_launches * args.steps
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
        "higher_is_better": True, "scaling": "strong" if wl.total else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": config_dict(F, wl),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1),
                     "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic, "traffic_source": traffic_src,
                     "traffic_over_algorithmic": (None if traffic is None
                                                  else round(traffic / bytes_pl, 3)),
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": bytes_pl,
                     "note": "algorithmic bytes per SURVEY.md 8d (unfused); fusion can make "
                             "achieved exceed DRAM traffic",
                     "compute": compute},
        "kernels": kernels,
        "stage_ms_per_step": {k: round(v, 4) for k, v in stage_ms.items()},
        "stage_note": "stage times from opcfe_front_end_profiled (stages back to back); the "
                      "timed step runs the same launches on one stream (opcfe_front_end)",
        "frame_hbm_frac": round(ab["frame_total"] * F / (max_ms / args.steps / 1e3) / 1e9 / peak, 4),
        "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": launches,
        "parity": parity, "strict": strict, "mixed": mixed, "distributed": dist_info,
        "clocks": clk.summary(), "n_tri_per_frame": T,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--frames", type=int, default=None,
                    help="frames per GPU per step (default: the workload's; C5: 512 / N)")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="C4",
                    help="BASELINE.json config (C4 = the metric's config, the default line)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-e2e-files", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e-dropin", action="store_true")
    ap.add_argument("--share-gpus", action="store_true",
                    help="dry run of the multi-rank path on fewer GPUs than ranks: rank r uses "
                         "GPU LOCAL_RANK %% device_count, gloo for the timing collectives "
                         "(plumbing check, NOT a scaling measurement)")
    ap.add_argument("--no-strict", action="store_true",
                    help="skip the strict (fp64 reference chain) and mixed-precision device "
                         "and e2e legs")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    wl = WORKLOADS[args.workload]
    if args.frames is None:
        args.frames = wl.frames
    if args.impl == "reference":
        return run_reference(args, rank, world, wl)
    if world > 1:
        import torch.distributed as dist
        import torch
        gpu = gpu_index(local_rank, args)
        torch.cuda.set_device(gpu)
        # NCCL refuses two ranks on one device: the shared-GPU dry run uses gloo (the only
        # collectives are the barrier and the max-over-ranks of a scalar)
        backend = os.environ.get("OPCFE_DIST_BACKEND") or ("gloo" if args.share_gpus else "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
        else:
            dist.init_process_group(backend)
    try:
        return run_ours(args, rank, world, local_rank, wl)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
