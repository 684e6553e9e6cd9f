import sys
import numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/dev'); sys.path.insert(0, '/root/repo/tests')
from stress_diag_gen import gen
import paper_2007_12065_b200 as fe
for seed in [int(a) for a in sys.argv[1:]]:
    frames, lap, bil, l_max = gen(seed)
    if lap is None or lap.kernel_size != 3: print(seed, 'skip', lap); continue
    x = frames[0]
    for L in (2, 3):
        fused = np.asarray(fe.laplacian_filter_opc(x, fe.LaplacianParams(lap.lam, 3, L)))
        cur = x
        for _ in range(L):
            cur = np.asarray(fe.laplacian_filter_opc(cur, fe.LaplacianParams(lap.lam, 3, 1)))
        d = (fused.view(np.uint32) != cur.view(np.uint32)).any(axis=2)
        idx = np.argwhere(d)
        print(seed, 'L', L, 'shape', x.shape, 'diff points', len(idx), idx[:6].tolist())
        for u, v in idx[:2]:
            print('   fused', fused[u, v].tolist(), 'chain', cur[u, v].tolist(), 'nan nbhd',
                  np.isnan(x[max(0,u-1):u+2, max(0,v-1):v+2, 0]).astype(int).tolist(), 'row in strip', u % 8, 'col', v % 32)
