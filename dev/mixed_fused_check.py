"""The mixed front end's fused FC data (OPCFE_MIXED_FUSED_FC=1, iteration 1 from the f64
grid) against the separate FC pass (=0): outputs must be bit-identical.  Runs both in
subprocesses (the switch is read at library load); C4, C2 and a NaN-holed odd-M frame."""
import os
import subprocess
import sys
import tempfile

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2007_12065_b200 as fe
rng = np.random.default_rng(3)
hole = fe.synthetic.room_scene(n=301, noise=0.002, seed=5)[:, :300].copy()
hole[rng.random(hole.shape[:2]) < 0.1] = np.nan
out = {}
for name, opc, bil in [("C4", fe.synthetic.config_c4(), (0.1, 0.15, 3, 5)),
                       ("C2", fe.synthetic.config_c2(), (0.1, 0.15, 5, 2)),
                       ("hole", hole, (0.05, 0.2, 3, 3))]:
    M, N = opc.shape[:2]
    eng = fe.FrontEnd(M, N, 1, laplacian=fe.LaplacianParams(1.0, 3, 3),
                      bilateral=fe.BilateralParams(*bil), src_dtype=torch.float64, precision="mixed")
    res = eng.run(torch.from_numpy(opc).cuda().unsqueeze(0))
    T = res.n_tri[0]
    out[name] = res.normals[0, :T].cpu().numpy()
    out[name + "_launches"] = np.array(eng.kernel_launches)
np.savez(sys.argv[2], **out)
'''
res = {}
for v in ("0", "1"):
    path = os.path.join(tempfile.mkdtemp(), f"m{v}.npz")
    r = subprocess.run([sys.executable, "-c", CHILD, REPO, path], env=dict(os.environ, OPCFE_MIXED_FUSED_FC=v),
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    res[v] = np.load(path)
for k in ("C4", "C2", "hole"):
    a, b = res["0"][k], res["1"][k]
    same = a.shape == b.shape and np.array_equal(np.isnan(a), np.isnan(b)) and \
        np.array_equal(np.nan_to_num(a), np.nan_to_num(b))
    d = np.nanmax(np.abs(a - b)) if a.shape == b.shape else None
    print(k, "bit-identical" if same else f"DIFFER max {d}", "launches",
          int(res["0"][k + "_launches"]), int(res["1"][k + "_launches"]))
