import numpy as np
import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import conftest
import paper_2007_12065_b200 as fe
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

