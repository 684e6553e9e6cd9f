"""Precision "mixed" under the randomised sweeps: the drop-in seeds of
test_gpu_parity.test_drop_in_api_randomised (incl. seed 26, a fast-mode 2.2e-5 case) and
200 random clouds of test_gpu_vs_reference.test_mixed_front_end_vs_stock_reference."""
import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import test_gpu_parity as T
import test_gpu_vs_reference as R
import paper_2007_12065_b200 as fe

fe.smoothing.set_precision('mixed')
bad = []
for seed in range(12, 112):
    try:
        T.test_drop_in_api_randomised(fe, seed)
    except Exception as e:
        bad.append(('dropin', seed, repr(e)[:200]))
ref = R.ref.__wrapped__()
for seed in range(12, 212):
    try:
        R.test_mixed_front_end_vs_stock_reference(fe, ref, seed)
    except Exception as e:
        bad.append(('frontend', seed, repr(e)[:200]))
print('mixed stress failures', len(bad)); print(bad[:10])
