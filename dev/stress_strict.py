"""500 seeds of the randomised strict-chain test (tests/test_gpu_strict.py) -- DESIGN.md 2."""
import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import test_gpu_strict as T
import paper_2007_12065_b200 as fe
bad = []
for seed in range(24, 524):
    try:
        T.test_strict_front_end_randomised(fe, seed)
    except Exception as e:
        bad.append((seed, repr(e)[:200]))
print('strict stress: 500 seeds, failures', len(bad)); print(bad[:10])
