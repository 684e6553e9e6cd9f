"""Diagnose the worst strict-chain normal (seed 329 of dev/stress_strict.py): per-iteration
error of the strict bilateral vs the C oracle on identical inputs, and the conditioning
(sum of weights / |acc|) of the worst triangle."""
import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from oracle import c_oracle
import paper_2007_12065_b200 as fe
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 329
rng = np.random.default_rng(5000 + seed)
M, N = int(rng.integers(3, 150)), int(rng.integers(3, 150))
F = int(rng.integers(1, 4))
frames = []
for _ in range(F):
    u, v = np.meshgrid(np.arange(M, dtype=float), np.arange(N, dtype=float), indexing="ij")
    s = rng.uniform(0.002, 0.05)
    opc = np.stack([v * s, -u * s, rng.normal(0, 0.01, (M, N)) + 0.2 * np.sin(np.arange(N) / 9.0)[None, :]], axis=2)
    opc += rng.normal(scale=rng.uniform(0, 0.004), size=opc.shape)
    for a, b in rng.integers(0, [max(1, M - 1), max(1, N - 1)], size=(int(rng.integers(0, 6)), 2)):
        opc[a, min(b + 1, N - 1)] = opc[a, b]
    opc[rng.random((M, N)) < rng.uniform(0, 0.4)] = np.nan
    if rng.random() < 0.5:
        opc[int(rng.integers(0, M)), int(rng.integers(0, N)), 1] = np.nan
    frames.append(opc)
k_lap = int(rng.choice([3, 3, 5, 7, 9, 11, 13]))
lap = (float(rng.uniform(0.3, 1.0)), k_lap, int(rng.integers(1, 7))) if rng.random() < 0.85 and min(M, N) >= k_lap else None
k_bil = int(rng.choice([3, 3, 3, 5, 7, 11, 13]))
bil = (float(rng.uniform(0.02, 0.3)), float(rng.uniform(0.05, 0.5)), k_bil, int(rng.integers(1, 4))) if rng.random() < 0.75 else None
print("config", M, N, F, lap, bil)
for f in range(F):
    sm = c_oracle.laplacian_filter(frames[f], *lap) if lap else frames[f]
    cen, nrm = c_oracle.compute_fc_triangle_data(sm)
    cur_ref = nrm
    for it in range(bil[3]):
        nxt_ref = c_oracle.bilateral_iterate(cen, cur_ref, bil[0], bil[1], bil[2], 1)
        nxt_gpu = fe._kernels.bilateral_iterate(cen, cur_ref, bil[0], bil[1], bil[2], 1)
        d = np.linalg.norm((nxt_gpu - nxt_ref).reshape(-1, 3), axis=1)
        d = np.nan_to_num(d)
        i = int(np.argmax(d))
        print(f"frame {f} it {it + 1}: one-step error on identical input max {d.max():.3e} at {i}")
        cur_ref = nxt_ref
    full_gpu = fe._kernels.bilateral_iterate(cen, nrm, bil[0], bil[1], bil[2], bil[3])
    d = np.nan_to_num(np.linalg.norm((full_gpu - cur_ref).reshape(-1, 3), axis=1))
    print(f"frame {f}: chained {bil[3]} iterations max {d.max():.3e}")
