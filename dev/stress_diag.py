import sys
import numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import conftest
import test_gpu_parity as T
import paper_2007_12065_b200 as fe
from oracle import c_oracle

def gen(seed):
    rng = np.random.default_rng(1000 + seed)
    M, N = int(rng.integers(3, 170)), int(rng.integers(3, 170))
    F = int(rng.integers(1, 4))
    frames = []
    for f in range(F):
        opc = conftest.grid_opc(M, N) * rng.uniform(0.002, 0.05)
        opc[..., 2] = rng.normal(0, 0.01, (M, N)) + 0.2 * np.sin(np.arange(N) / 9.0)[None, :]
        opc += rng.normal(scale=rng.uniform(0, 0.004), size=opc.shape)
        for u, v in rng.integers(0, [max(1, M - 1), max(1, N - 1)], size=(int(rng.integers(0, 6)), 2)):
            opc[u, min(v + 1, N - 1)] = opc[u, v]
        opc[rng.random((M, N)) < rng.uniform(0, 0.4)] = np.nan
        frames.append(opc.astype(np.float32))
    k_lap = int(rng.choice([3, 3, 3, 5, 7]))
    lap = fe.LaplacianParams(float(rng.uniform(0.3, 1.0)), k_lap, int(rng.integers(1, 7))) \
        if rng.random() < 0.85 and min(M, N) >= k_lap else None
    k_bil = int(rng.choice([3, 3, 3, 5, 7]))
    bil = fe.BilateralParams(float(rng.uniform(0.02, 0.3)), float(rng.uniform(0.08, 0.5)), k_bil,
                             int(rng.integers(1, 4))) if rng.random() < 0.75 else None
    l_max = float(rng.uniform(0.001, 0.05)) if rng.random() < 0.5 else None
    return frames, lap, bil, l_max

seed = int(sys.argv[1])
frames, lap, bil, l_max = gen(seed)
print('lap', lap, 'bil', bil, 'l_max', l_max, 'shape', frames[0].shape, 'F', len(frames))
F = len(frames); M, N = frames[0].shape[:2]
_, res = T._engine_run(fe, np.stack(frames), lap, bil, l_max, frames=F)
f = 0
sm = res.points[f].cpu().numpy().astype(np.float64)
if lap is not None:
    ref = c_oracle.laplacian_filter(frames[f].astype(np.float64), lap.lam, lap.kernel_size, lap.iterations)
    err = np.linalg.norm(sm - ref, axis=2)
    err[np.isnan(err)] = 0
    idx = np.argwhere(err > 1e-6)
    print('lap bad points', len(idx), idx[:10].tolist(), 'max', err.max())
    for u, v in idx[:3]:
        print(' ', u, v, 'gpu', sm[u, v], 'ref', ref[u, v], 'in', frames[f][u, v])
        print('   nbhd nan', np.isnan(frames[f][max(0,u-1):u+2, max(0,v-1):v+2, 0]).astype(int).tolist())
        print('   nbhd', frames[f][max(0,u-1):u+2, max(0,v-1):v+2].tolist())
if bil is not None:
    from paper_2007_12065_b200 import _ops
    grid, _ = _ops.stage_in(res.points[f].contiguous(), want_points=True, want_mask=False)
    cen, nrm = c_oracle.compute_fc_triangle_data(sm)
    args = (bil.sigma_length, bil.sigma_angle, bil.kernel_size, 1)
    out = _ops.bilateral(1, M, N, *args, grid=grid, fc_normals=None)
    g = out[0, :, :6 * (N - 1)].reshape(M - 1, N - 1, 2, 3).cpu().numpy().astype(np.float64)
    r = c_oracle.bilateral_iterate(cen, nrm, *args)
    gn, rn = np.isnan(g).any(-1), np.isnan(r).any(-1)
    bad = np.argwhere(gn != rn)
    print('bil iter1 nan mismatches', len(bad), bad[:5].tolist())
    for u, v, k in bad[:3]:
        print('  gpu', g[u, v, k], 'ref', r[u, v, k], 'fc normal', nrm[u, v, k], 'centroid', cen[u, v, k])
        print('  quad pts', sm[u:u+2, v:v+2].tolist())
