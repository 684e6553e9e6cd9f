"""How far a MIXED chain -- strict (fp64, bit-exact) Laplacian and FC data, then the fp32
bilateral on those exact FC arrays -- lands from the reference's fp64 chain (our strict
chain, which matches it to ~4e-14): C4 frame + the chain goldens."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2007_12065_b200 as fe  # noqa: E402
from paper_2007_12065_b200 import smoothing  # noqa: E402

def chain(opc, lap, bil, mode):
    sm = fe.laplacian_filter_opc(opc, fe.LaplacianParams(*lap), precision="strict")
    mesh = fe.mesh_from_opc(sm)
    if mode == "strict":
        return fe.bilateral_filter_opc(sm, fe.BilateralParams(*bil), mesh.trimap, precision="strict")
    cen, nrm = fe.compute_fc_triangle_data(sm)            # fp64, bit-exact
    smoothing.set_precision("fast")
    try:
        flat = fe._kernels.bilateral_iterate(cen, nrm, *bil).reshape(-1, 3)
    finally:
        smoothing.set_precision("auto")
    tm = mesh.trimap
    out = np.empty((int((tm >= 0).sum()), 3))
    out[tm[tm >= 0]] = flat[tm >= 0]
    return out

cases = [("C4", fe.synthetic.config_c4(), (1.0, 3, 10), (0.1, 0.15, 3, 5)),
         ("C2", fe.synthetic.config_c2(), (1.0, 3, 3), (0.1, 0.15, 3, 2))]
z = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "chain.npz"))
for name in ("room72", "c2crop", "lidar_bil", "far"):
    cases.append((name, z[f"{name}/opc"], tuple(z[f"{name}/lap"]), tuple(z[f"{name}/bil"])))
for name, opc, lap, bil in cases:
    lap = (float(lap[0]), int(lap[1]), int(lap[2]))
    bil = (float(bil[0]), float(bil[1]), int(bil[2]), int(bil[3]))
    s = chain(opc, lap, bil, "strict")
    m = chain(opc, lap, bil, "mixed")
    ok = ~np.isnan(s).any(1)
    assert np.array_equal(ok, ~np.isnan(m).any(1))
    e = np.linalg.norm(m[ok] - s[ok], axis=1)
    print(f"{name}: n={ok.sum()} max={e.max():.2e} p99.9={np.quantile(e, 0.999):.2e} "
          f">1e-5: {(e > 1e-5).sum()}")
