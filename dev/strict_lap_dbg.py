import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2007_12065_b200 as fe
base = fe.synthetic.config_c2()
for rep in range(3):
    g = fe.laplacian_filter_opc(base, fe.LaplacianParams(1.0, 3, 1), precision="strict")
    nan = np.argwhere(np.isnan(g[..., 0]) & ~np.isnan(base[..., 0]))
    print(rep, len(nan), [(int(u), int(v), int(u % 8), g[u, v, 1], g[u, v, 2]) for u, v in nan[:8]])
