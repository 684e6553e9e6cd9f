"""One mixed-precision C4 step (16 frames, lap 10 + bil 5) for ncu launch lists."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_12065_b200 as fe  # noqa: E402

eng = fe.FrontEnd(1080, 1920, 16, laplacian=fe.LaplacianParams(1.0, 3, 10),
                  bilateral=fe.BilateralParams(0.1, 0.15, 3, 5), src_dtype=torch.float64,
                  graph=False, precision=os.environ.get("PREC", "mixed"))
eng.src.copy_(torch.from_numpy(fe.synthetic.config_c4()).cuda().expand_as(eng.src))
for _ in range(2):
    eng.run(eng.src)
torch.cuda.synchronize()
print("ok")
