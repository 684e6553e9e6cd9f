"""Precision "mixed" against strict (the reference's chain to ~4e-14) on whole frames:
smoothed-vertex deviation (m, relative) and final-normal deviation.  C4 and C2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2007_12065_b200 as fe  # noqa: E402

for name, opc, lap, bil in [("C4", fe.synthetic.config_c4(), (1.0, 3, 10), (0.1, 0.15, 3, 5)),
                            ("C2", fe.synthetic.config_c2(), (1.0, 3, 3), (0.1, 0.15, 3, 2))]:
    M, N = opc.shape[:2]
    out = {}
    for prec in ("strict", "mixed"):
        eng = fe.FrontEnd(M, N, 1, laplacian=fe.LaplacianParams(*lap),
                          bilateral=fe.BilateralParams(*bil), src_dtype=torch.float64, graph=False,
                          precision=prec)
        res = eng.run(torch.from_numpy(opc).cuda().unsqueeze(0))
        T = res.n_tri[0]
        out[prec] = (res.points[0].cpu().numpy(), res.trimap[0].cpu().numpy(),
                     res.normals[0, :T].cpu().numpy().astype(np.float64))
    (sp, st, sn), (mp, mt, mn) = out["strict"], out["mixed"]
    ok = np.isfinite(sp).all(2)
    dv = np.linalg.norm(mp[ok] - sp[ok], axis=1)
    rel = dv / np.linalg.norm(sp[ok], axis=1)
    good = ~np.isnan(sn).any(1)
    dn = np.linalg.norm(mn[good] - sn[good], axis=1)
    print(name, "topology", np.array_equal(st, mt), "vertices: max %.3g m, rel max %.3g, bit-exact %.4f"
          % (dv.max(), rel.max(), (dv == 0).mean()),
          "normals: max %.3g p99.9 %.3g n>1e-5 %d" % (dn.max(), np.quantile(dn, 0.999), (dn > 1e-5).sum()))
