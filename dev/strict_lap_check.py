"""Strict Laplacian (one pass, k = 3) against the C oracle on a full-size cloud: mismatch
count and the first mismatching positions (tile coordinates)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2007_12065_b200 as fe  # noqa: E402
from oracle import c_oracle  # noqa: E402

base = fe.synthetic.config_c2()
for it in (1, 2, 3):
    g = fe.laplacian_filter_opc(base, fe.LaplacianParams(1.0, 3, it), precision="strict")
    r = c_oracle.laplacian_filter(base, 1.0, 3, it)
    bad = ~((g == r) | (np.isnan(g) & np.isnan(r))).all(axis=2)
    idx = np.argwhere(bad)
    print(f"iters {it}: {len(idx)} mismatching points of {bad.size}")
    for u, v in idx[:8]:
        print("  u v", u, v, "tile", (u % 8, v % 32), g[u, v], r[u, v], "centre nan", np.isnan(base[u, v]).any(),
              "nbr nan", np.isnan(base[max(u-1,0):u+2, max(v-1,0):v+2]).any(axis=2).sum())

# which pair is off at the first mismatching point of one pass
g = fe.laplacian_filter_opc(base, fe.LaplacianParams(1.0, 3, 1), precision="strict")
r = c_oracle.laplacian_filter(base, 1.0, 3, 1)
bad = np.argwhere(~((g == r) | (np.isnan(g) & np.isnan(r))).all(axis=2))
u, v = bad[0]
p = base[u, v]
terms = []
for du in (-1, 0, 1):
    for dv in (-1, 0, 1):
        if du == 0 and dv == 0:
            continue
        d = base[u + du, v + dv] - p
        dist = np.sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2])
        terms.append(((du, dv), d / dist if dist > 0 else np.zeros(3), 1 / dist if dist > 0 else 0.0))
def combine(ts):
    a = np.zeros(3); w = 0.0
    for _, dw, ww in ts:
        a = a + dw; w = w + ww
    return p + (1.0 / w) * a if w > 0 else p
print("point", u, v, "gpu", g[u, v], "ref", r[u, v], "restated", combine(terms))
for i in range(8):
    alt = combine(terms[:i] + terms[i + 1:])
    print("  without", terms[i][0], np.abs(alt - g[u, v]).max())
for i in range(8):
    t2 = list(terms); t2[i] = (t2[i][0], -t2[i][1], t2[i][2])
    print("  negated", terms[i][0], np.abs(combine(t2) - g[u, v]).max())
