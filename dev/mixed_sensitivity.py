"""How much the reference's own fp64 bilateral moves when its input normals / centroids are
rounded to fp32 (C oracle), for the random clouds of test_gpu_vs_reference: the floor
under any fp32 bilateral (precision "mixed").  Usage: mixed_sensitivity.py SEED..."""
import sys
import numpy as np
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import test_gpu_vs_reference as R
from oracle import c_oracle as co
for seed in [int(s) for s in sys.argv[1:]]:
    rng = np.random.default_rng(9300 + seed)
    opc = R.random_cloud(rng)
    lap = (float(rng.uniform(0.2, 1.0)), 3, int(rng.integers(1, 6)))
    bil = (float(rng.uniform(0.02, 0.3)), float(rng.uniform(0.05, 0.5)), int(rng.choice([3, 5, 7])), int(rng.integers(1, 4)))
    sm = co.laplacian_filter(opc, *lap)
    cen, nrm = co.compute_fc_triangle_data(sm)
    ref = co.bilateral_iterate(cen, nrm, *bil)
    ok = ~np.isnan(ref).any(-1)
    r32 = lambda a: a.astype(np.float32).astype(np.float64)
    mu = np.nanmean(cen.reshape(-1,3), axis=0)
    def err(c, n):
        o = co.bilateral_iterate(c, n, *bil)
        return np.linalg.norm((o-ref)[ok], axis=-1).max()
    print(seed, 'offset', mu.round(2), 'n32', err(cen, r32(nrm)), 'c32', err(r32(cen), nrm),
          'both', err(r32(cen), r32(nrm)), 'c32 shifted', err(r32(cen-mu), nrm))
