import sys
import numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/dev'); sys.path.insert(0, '/root/repo/tests')
from stress_diag_gen import gen
import test_gpu_parity as T
import paper_2007_12065_b200 as fe
from paper_2007_12065_b200 import _ops
from oracle import c_oracle
seed = int(sys.argv[1])
frames, lap, bil, l_max = gen(seed)
print('lap', lap, 'bil', bil, 'shape', frames[0].shape, 'F', len(frames))
F = len(frames); M, N = frames[0].shape[:2]
_, res = T._engine_run(fe, np.stack(frames), lap, bil, l_max, frames=F)
for f in range(F):
    sm = res.points[f].cpu().numpy().astype(np.float64)
    grid, _ = _ops.stage_in(res.points[f].contiguous(), want_points=True, want_mask=False)
    cen, ref_in = c_oracle.compute_fc_triangle_data(sm)
    prev = None
    args = (bil.sigma_length, bil.sigma_angle, bil.kernel_size, 1)
    for it in range(1, bil.iterations + 1):
        ref = c_oracle.bilateral_iterate(cen, ref_in, *args)
        out = _ops.bilateral(1, M, N, *args, grid=grid, fc_normals=prev)
        g = out[0, :, :6 * (N - 1)].reshape(M - 1, N - 1, 2, 3).cpu().numpy().astype(np.float64)
        e = np.linalg.norm(g - ref, axis=-1); e[np.isnan(e)] = 0
        i = np.unravel_index(np.argmax(e), e.shape)
        print('frame', f, 'it', it, 'max err', e.max(), 'at', i, 'n>1e-5', int((e > 1e-5).sum()))
        if e.max() > 1e-5:
            u, v, k = i
            print('   gpu', g[i], 'ref', ref[i], 'in normal', ref_in[i])
            h = bil.kernel_size // 2
            win = ref_in[max(0,u-h):u+h+1, max(0,v-h):v+h+1]
            cw = cen[max(0,u-h):u+h+1, max(0,v-h):v+h+1]
            A = 1/(2*bil.sigma_length**2); B = 1/(2*bil.sigma_angle**2)
            dc = ((cw - cen[i])**2).sum(-1); dn = ((win - ref_in[i])**2).sum(-1)
            wts = np.exp(-dc*A - dn*B)
            print('   weights', np.round(np.sort(wts[np.isfinite(wts)].ravel())[::-1][:8], 8), 'sum', np.nansum(wts))
            acc = np.nansum(wts[..., None] * np.nan_to_num(win), axis=(0,1,2))
            print('   |acc|', np.linalg.norm(acc))
        ref_in = g; prev = out
