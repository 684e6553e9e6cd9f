"""Determinism of the strict Laplacian (one pass, k = 3) on C2: mismatches vs the oracle
over repeated runs (positions as (u, v, ty, tx, blockIdx.y, blockIdx.x))."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2007_12065_b200 as fe  # noqa: E402
from oracle import c_oracle  # noqa: E402

base = fe.synthetic.config_c2()
r = c_oracle.laplacian_filter(base, 1.0, 3, 1)
for rep in range(4):
    g = fe.laplacian_filter_opc(base, fe.LaplacianParams(1.0, 3, 1), precision="strict")
    bad = np.argwhere(~((g == r) | (np.isnan(g) & np.isnan(r))).all(axis=2))
    print(rep, len(bad), [(int(u), int(v), int(u % 8), int(v % 32), int(u // 8), int(v // 32)) for u, v in bad[:6]])
