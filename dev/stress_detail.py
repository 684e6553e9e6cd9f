import sys, traceback
import numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import test_gpu_parity as T
import paper_2007_12065_b200 as fe
for seed in [int(s) for s in sys.argv[1:]]:
    rng = np.random.default_rng(1000 + seed)
    M, N = int(rng.integers(3, 170)), int(rng.integers(3, 170))
    F = int(rng.integers(1, 4))
    print('seed', seed, 'M N F', M, N, F)
    try:
        T.test_front_end_randomised(fe, seed)
        print('  ok')
    except Exception:
        tb = traceback.format_exc().splitlines()
        print('\n'.join(tb[-12:]))
