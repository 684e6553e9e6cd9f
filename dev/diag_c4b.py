"""Scratch diagnostic: bilateral error growth per iteration at C4."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2007_12065_b200 as fe
from oracle import c_oracle

opc = fe.synthetic.config_c4()
M, N = opc.shape[:2]
lap = fe.LaplacianParams(1.0, 3, 10)
eng = fe.FrontEnd(M, N, 1, laplacian=lap, bilateral=None)
res = eng.run(torch.from_numpy(opc).float().cuda().unsqueeze(0))
torch.cuda.synchronize()
grid = eng.grid.clone()
sm = res.points[0].cpu().numpy().astype(np.float64)
tris, trimap, he = c_oracle.triangulate(sm)
T = len(tris)
cen, nrm = c_oracle.compute_fc_triangle_data(sm)
tm = torch.from_numpy(trimap).cuda().unsqueeze(0)
from paper_2007_12065_b200 import _ops
cur = nrm
for it in range(1, 6):
    ref_fc = c_oracle.bilateral_iterate(cen, nrm, 0.1, 0.15, 3, it)
    ref = c_oracle.gather(ref_fc, trimap, T)
    g = _ops.bilateral(1, M, N, 0.1, 0.15, 3, it, grid=grid, trimap=tm, out_rows=T)[0].cpu().numpy()
    err = np.linalg.norm(g - ref, axis=1)
    err[~np.isfinite(err)] = 0
    t = int(np.argmax(err))
    gid = np.nonzero(trimap == t)[0][0]
    q, k = divmod(gid, 2); u, v = divmod(q, N - 1)
    print(f"iters={it}: max err {err.max():.2e} at (u,v,k)=({u},{v},{k}); over1e-5={int((err>1e-5).sum())}; p99.99={np.quantile(err,0.9999):.2e}")
    # one-step error from the oracle's previous normals (isolates per-iteration error)
