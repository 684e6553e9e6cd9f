"""One strict Laplacian pass chain (C4, 16 frames, k = 3, 2 passes) for ncu captures of the
strict Laplacian kernels (OPCFE_LAP64_TMA=0 selects the per-thread staging)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_12065_b200 as fe
from paper_2007_12065_b200 import _ops
x = torch.from_numpy(fe.synthetic.config_c4()).cuda().unsqueeze(0).expand(16, -1, -1, -1).contiguous()
for _ in range(2):
    y = _ops.laplacian_f64(x, 1.0, 3, 2)
torch.cuda.synchronize()
print("ok", tuple(y.shape))
