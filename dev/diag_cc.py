"""Scratch: GPU same-label components vs scipy connected_components on the golden meshes."""
import sys
import numpy as np
import torch
from scipy.sparse import coo_matrix
from scipy.sparse.csgraph import connected_components
sys.path.insert(0, ".")
from paper_2007_12065_b200 import _ops

z = np.load("tests/golden/segments.npz")
for sc in ("room", "frag"):
    tris, he, groups = z[sc + "_triangles"], z[sc + "_halfedges"], z[sc + "_groups"]
    n = len(tris)
    t = np.repeat(np.arange(n), 3); u = he // 3; ok = he >= 0
    t, u = t[ok], u[ok]
    same = (groups[t] == groups[u]) & (groups[t] != 255)
    A = coo_matrix((np.ones(same.sum()), (t[same], u[same])), shape=(n, n))
    _, lab = connected_components(A, directed=False)
    # expected root = min index of the component
    mins = {}
    for i in range(n):
        mins.setdefault(lab[i], i)
    exp = np.array([mins[lab[i]] if groups[i] != 255 else -1 for i in range(n)])
    for rep in range(3):
        comp, size = _ops.segment_components(torch.from_numpy(he).cuda(), torch.from_numpy(groups).cuda())
        c = comp.cpu().numpy()
        bad = np.nonzero(c != exp)[0]
        print(sc, rep, "mismatch", len(bad), bad[:10], c[bad[:10]], exp[bad[:10]])
