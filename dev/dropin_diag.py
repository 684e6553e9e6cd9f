import sys
import numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import conftest
import paper_2007_12065_b200 as fe
from oracle import flatpoly_oracle as fo
seed = int(sys.argv[1])
rng = np.random.default_rng(500 + seed)
M, N = int(rng.integers(5, 90)), int(rng.integers(5, 90))
opc = conftest.grid_opc(M, N) * rng.uniform(0.003, 0.03)
opc[..., 2] = rng.normal(0, 0.005, (M, N))
opc += rng.normal(scale=rng.uniform(0, 0.003), size=opc.shape)
opc[rng.integers(0, M), :] = opc[rng.integers(0, M), :]
opc[rng.random((M, N)) < rng.uniform(0, 0.3)] = np.nan
k = int(rng.choice([3, 5]))
lp = fe.LaplacianParams(float(rng.uniform(0.2, 1.0)), k, int(rng.integers(1, 5)))
sm = fe.laplacian_filter_opc(opc, lp)
bp = fe.BilateralParams(float(rng.uniform(0.03, 0.2)), float(rng.uniform(0.1, 0.4)), int(rng.choice([3, 5])), 1)
print('shape', M, N, 'bil', bp)
cen, nrm = fo.compute_fc_triangle_data(sm)
g = np.asarray(fe._kernels.bilateral_iterate(cen, nrm, bp.sigma_length, bp.sigma_angle, bp.kernel_size, 1))
r = fo.bilateral_iterate(cen, nrm, bp.sigma_length, bp.sigma_angle, bp.kernel_size, 1)
e = np.linalg.norm(g - r, axis=-1); e[np.isnan(e)] = 0
i = np.unravel_index(np.argmax(e), e.shape)
print('max err', e.max(), 'at', i)
u, v, kk = i; h = bp.kernel_size // 2
A = 1 / (2 * bp.sigma_length**2); B = 1 / (2 * bp.sigma_angle**2)
acc = np.zeros(3); wsum = 0
for du in range(-h, h + 1):
    for dv in range(-h, h + 1):
        for k2 in range(2):
            if du == 0 and dv == 0 and k2 == kk: continue
            uu, vv = u + du, v + dv
            if not (0 <= uu < cen.shape[0] and 0 <= vv < cen.shape[1]): continue
            n2 = nrm[uu, vv, k2]
            if np.isnan(n2).any(): continue
            w = np.exp(-A * ((cen[uu, vv, k2] - cen[i])**2).sum() - B * ((n2 - nrm[i])**2).sum())
            acc += w * n2; wsum += w
print('wsum', wsum, '|acc|', np.linalg.norm(acc), 'kappa', wsum / np.linalg.norm(acc), 'centroid', cen[i], 'A', A, 'B', B)
