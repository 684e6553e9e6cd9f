"""The STOCK reference's organized chain (pipeline.py:125-134) with libopcfe plugged into
its own kernel switch (integration/: FLATPOLY_CUDA=1), NumPy float64 in and out, one C4
frame per call: per-frame wall time.  Usage: python dev/plugin_e2e.py [strict|fast]"""
import json
import os
import subprocess
import sys
import tempfile

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
mode = sys.argv[1] if len(sys.argv) > 1 else "strict"
dest = tempfile.mkdtemp(prefix="flatpoly_cuda_")
subprocess.run([sys.executable, os.path.join(REPO, "integration", "install.py"), dest], check=True,
               stdout=subprocess.DEVNULL)
sys.path.insert(0, REPO)
import numpy as np  # noqa: E402

from paper_2007_12065_b200 import synthetic  # noqa: E402

frame_path = os.path.join(dest, "frame.npy")
np.save(frame_path, synthetic.config_c4())
code = r'''
import json, sys, time
import numpy as np
from flatpoly import _kernels, mesh, smoothing
assert _kernels.ACTIVE == "cuda", _kernels.ACTIVE
opc = np.load(sys.argv[1])
lp, bp = smoothing.LaplacianParams(1.0, 3, 10), smoothing.BilateralParams(0.1, 0.15, 3, 5)
def one():
    sm = smoothing.laplacian_filter_opc(opc, lp)
    m = mesh.mesh_from_opc(sm)
    m.normals = smoothing.bilateral_filter_opc(sm, bp, m.trimap)
    return sm, m
sm, m = one(); sm, m = one()
t = time.perf_counter()
n = 5
for _ in range(n):
    sm, m = one()
dt = (time.perf_counter() - t) / n
print(json.dumps({"frames_per_s": 1.0 / dt, "ms_per_frame": 1e3 * dt, "triangles": int(m.num_triangles)}))
if len(sys.argv) > 2:
    import cProfile, pstats
    pr = cProfile.Profile(); pr.enable(); one(); pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(12)
'''
env = dict(os.environ, FLATPOLY_CUDA="1" if mode == "strict" else "fast",
           OPCFE_LIB=os.path.join(REPO, "paper_2007_12065_b200", "lib", "libopcfe.so"),
           PYTHONPATH=os.pathsep.join([dest, os.path.join(REPO, "tests", "golden", "_stubs")]))
r = subprocess.run([sys.executable, "-c", code, frame_path] + sys.argv[2:3], env=env, capture_output=True,
                   text=True, cwd=dest)
print(mode, r.stdout.strip() or r.stderr[-2000:])
