import sys
import numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/dev'); sys.path.insert(0, '/root/repo/tests')
from stress_diag_gen import gen
import paper_2007_12065_b200 as fe
from paper_2007_12065_b200 import _ops
from oracle import c_oracle
frames, lap, bil, l_max = gen(int(sys.argv[1]))
x = frames[0]
M, N = x.shape[:2]
cur = x.astype(np.float32)
pts = [(9,146),(9,147),(15,36),(16,36)]
for it in range(1, lap.iterations + 1):
    g = fe.laplacian_filter_opc(cur, fe.LaplacianParams(lap.lam, 3, 1))   # one GPU pass on cur
    r = c_oracle.laplacian_filter(cur.astype(np.float64), lap.lam, 3, 1)  # one fp64 pass on cur
    e = np.linalg.norm(np.asarray(g, np.float64) - r, axis=2); e[np.isnan(e)] = 0
    print(it, 'per-pass max abs err', e.max(), [ (p, np.asarray(g)[p].round(6).tolist(), r[p].round(6).tolist()) for p in pts[:2]])
    cur = np.asarray(g, dtype=np.float32)
# full chain fp32 GPU (6 passes, one launch) vs chaining single passes
full = fe.laplacian_filter_opc(x, fe.LaplacianParams(lap.lam, 3, lap.iterations))
print('fused vs chained single passes max diff', np.nanmax(np.abs(np.asarray(full) - cur)))
