"""Scratch diagnostic: bilateral error per launch and chained, for the kernel variant the
environment selects (OPCFE_BILATERAL_DOTN / _WS).  One JSON line per config.

per_iter: each launch vs one fp64 oracle iteration applied to the same fp32 input normals
chained:  the fused B-iteration output vs the fp64 B-iteration chain
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2007_12065_b200 as fe  # noqa: E402
from paper_2007_12065_b200 import _ops  # noqa: E402
from oracle import c_oracle  # noqa: E402


def run(name, opc, lap, bil):
    M, N = opc.shape[:2]
    Mq, Nq = M - 1, N - 1
    eng = fe.FrontEnd(M, N, 1, laplacian=lap, bilateral=bil)
    res = eng.run(torch.from_numpy(opc).float().cuda().unsqueeze(0))
    torch.cuda.synchronize()
    sm = res.points[0].cpu().numpy().astype(np.float64)
    T = int(res.n_tri[0])
    tris, trimap, _ = c_oracle.triangulate(sm)
    grid, _ = _ops.stage_in(res.points[0].contiguous(), want_points=True, want_mask=False)
    cen, ref_in = c_oracle.compute_fc_triangle_data(sm)
    nrm0 = ref_in
    args = (bil.sigma_length, bil.sigma_angle, bil.kernel_size, 1)
    prev = None
    per_iter = []
    for it in range(1, bil.iterations + 1):
        ref = c_oracle.bilateral_iterate(cen, ref_in, *args)
        out = _ops.bilateral(1, M, N, *args, grid=grid, fc_normals=prev)
        g = out[0, :, :6 * Nq].reshape(Mq, Nq, 2, 3).cpu().numpy().astype(np.float64)
        e = np.linalg.norm(g - ref, axis=-1)
        e = e[np.isfinite(e)]
        per_iter.append((float(e.max()), int((e > 1e-5).sum()), int((e > 1e-6).sum())))
        ref_in, prev = g, out
    full = c_oracle.bilateral_iterate(cen, nrm0, bil.sigma_length, bil.sigma_angle,
                                      bil.kernel_size, bil.iterations)
    err = np.linalg.norm(res.normals[0, :T].cpu().numpy() - c_oracle.gather(full, trimap, T), axis=1)
    err = err[np.isfinite(err)]
    print(json.dumps({
        "config": name, "variant": {k: v for k, v in os.environ.items() if k.startswith("OPCFE_")},
        "per_iter_max": [p[0] for p in per_iter], "per_iter_over_1e-5": [p[1] for p in per_iter],
        "per_iter_over_1e-6": [p[2] for p in per_iter],
        "chained_max": float(err.max()), "chained_over_1e-5": int((err > 1e-5).sum()),
        "chained_p9999": float(np.quantile(err, 0.9999)), "triangles": T}), flush=True)


syn = fe.synthetic
run("C1", syn.config_c1(), fe.LaplacianParams(1.0, 3, 1), fe.BilateralParams(0.1, 0.15, 3, 1))
run("C2", syn.config_c2(), fe.LaplacianParams(1.0, 3, 3), fe.BilateralParams(0.1, 0.15, 3, 2))
run("C4", syn.config_c4(), fe.LaplacianParams(1.0, 3, 10), fe.BilateralParams(0.1, 0.15, 3, 5))
run("C4-k5", syn.config_c4(), fe.LaplacianParams(1.0, 3, 10), fe.BilateralParams(0.1, 0.15, 5, 3))
run("C4-sa0.05", syn.config_c4(), fe.LaplacianParams(1.0, 3, 2), fe.BilateralParams(0.05, 0.05, 3, 3))
