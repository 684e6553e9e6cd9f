"""Where the drop-in API's time goes at C4 (one frame per call, NumPy f64 in / out):
per-call wall times, and the raw pageable / pinned copy bandwidth of this host."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2007_12065_b200 as fe  # noqa: E402


def bw(fn, nbytes, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t) / 1e9


n = 100 << 20
d = torch.empty(n, dtype=torch.uint8, device="cuda")
hp = torch.empty(n, dtype=torch.uint8, pin_memory=True)
print(f"pinned D2H {bw(lambda: hp.copy_(d), n):.1f} GB/s, pinned H2D {bw(lambda: d.copy_(hp), n):.1f} GB/s")
print(f"pageable D2H into a fresh array (.cpu()) {bw(lambda: d.cpu(), n):.1f} GB/s")
a = np.empty(n, dtype=np.uint8)
a[:] = 1
ta = torch.from_numpy(a)
print(f"pageable D2H into a touched array {bw(lambda: ta.copy_(d), n):.1f} GB/s")
print(f"pageable H2D from a touched array {bw(lambda: d.copy_(ta), n):.1f} GB/s")
print(f"np.empty + first touch {n * 5 / sum((lambda t0: (np.ones(n, np.uint8), time.perf_counter() - t0)[1])(time.perf_counter()) for _ in range(5)) / 1e9:.1f} GB/s")

frame = fe.synthetic.config_c4()
lp, bp = fe.LaplacianParams(1.0, 3, 10), fe.BilateralParams(0.1, 0.15, 3, 5)
for prec in ("strict", "fast"):
    for rep in range(3):
        t0 = time.perf_counter()
        sm = fe.laplacian_filter_opc(frame, lp, precision=prec)
        t1 = time.perf_counter()
        mesh = fe.mesh_from_opc(sm)
        t2 = time.perf_counter()
        mesh.normals = fe.bilateral_filter_opc(sm, bp, mesh.trimap, precision=prec)
        t3 = time.perf_counter()
        if rep:
            print(f"{prec}: laplacian {1e3*(t1-t0):.1f} ms, mesh_from_opc {1e3*(t2-t1):.1f} ms, "
                  f"bilateral {1e3*(t3-t2):.1f} ms, total {1e3*(t3-t0):.1f} ms")
import cProfile, pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
sm = fe.laplacian_filter_opc(frame, lp)
mesh = fe.mesh_from_opc(sm)
mesh.normals = fe.bilateral_filter_opc(sm, bp, mesh.trimap)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
