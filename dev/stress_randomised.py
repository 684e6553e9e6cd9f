import sys, traceback
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import test_gpu_parity as T
import paper_2007_12065_b200 as fe
fe.smoothing.set_precision('fast')   # the fp32 path under stress (test_gpu_parity's fixture)
bad = []
for seed in range(40, 340):
    try:
        T.test_front_end_randomised(fe, seed)
    except Exception as e:
        bad.append((seed, repr(e)[:200]))
for seed in range(12, 112):
    try:
        T.test_drop_in_api_randomised(fe, seed)
    except Exception as e:
        bad.append(('dropin', seed, repr(e)[:200]))
print('failures', len(bad)); print(bad[:10])
