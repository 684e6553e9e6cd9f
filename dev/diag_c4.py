"""Scratch diagnostic: worst bilateral errors at C4 and their conditioning."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2007_12065_b200 as fe
from oracle import c_oracle

opc = fe.synthetic.config_c4()
lap, bil = fe.LaplacianParams(1.0, 3, 10), fe.BilateralParams(0.1, 0.15, 3, 5)
M, N = opc.shape[:2]
eng = fe.FrontEnd(M, N, 1, laplacian=lap, bilateral=bil)
res = eng.run(torch.from_numpy(opc).float().cuda().unsqueeze(0))
torch.cuda.synchronize()
sm = res.points[0].cpu().numpy().astype(np.float64)
T = res.n_tri[0]
tris, trimap, he = c_oracle.triangulate(sm)
cen, nrm = c_oracle.compute_fc_triangle_data(sm)
prev = c_oracle.bilateral_iterate(cen, nrm, 0.1, 0.15, 3, 4)
last = c_oracle.bilateral_iterate(cen, prev, 0.1, 0.15, 3, 1)
ref = c_oracle.gather(last, trimap, T)
g = res.normals[0, :T].cpu().numpy()
err = np.linalg.norm(g - ref, axis=1)
err[~np.isfinite(err)] = 0
order = np.argsort(-err)[:12]
print("n over 1e-5:", int((err > 1e-5).sum()), "of", T, "max", err.max())
# conditioning |acc|/wsum at the last iteration for the worst triangles
inv = np.full(len(trimap), -1); inv[trimap[trimap >= 0]] = np.nonzero(trimap >= 0)[0]
Mq, Nq = M - 1, N - 1
P = prev.reshape(Mq, Nq, 2, 3); C = cen.reshape(Mq, Nq, 2, 3)
ic, isg = 1 / (2 * 0.1 ** 2), 1 / (2 * 0.15 ** 2)
for t in order:
    gid = inv[t]; q, k = divmod(gid, 2); u, v = divmod(q, Nq)
    acc = np.zeros(3); ws = 0.0
    for du in (-1, 0, 1):
        for dv in (-1, 0, 1):
            for kk in (0, 1):
                uu, vv = u + du, v + dv
                if (du, dv, kk) == (0, 0, k) or not (0 <= uu < Mq and 0 <= vv < Nq):
                    continue
                m = P[uu, vv, kk]
                if np.isnan(m).any():
                    continue
                w = np.exp(-np.sum((C[uu, vv, kk] - C[u, v, k]) ** 2) * ic - np.sum((m - P[u, v, k]) ** 2) * isg)
                acc += m * w; ws += w
    print(f"t={t} err={err[t]:.2e} |acc|/wsum={np.linalg.norm(acc)/ws:.4f} wsum={ws:.3e} (u,v,k)=({u},{v},{k})")
