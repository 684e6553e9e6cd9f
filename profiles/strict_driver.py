"""Drive the STRICT (fp64) -- or, with --precision mixed, the MIXED -- front end at C4 for
ncu captures (profiles/collect.sh): `--steps` batches of `--frames` 1080x1920 frames,
lap 10 + bil 5, eager launches."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2007_12065_b200 as fe  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=16)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--precision", default="strict", choices=("strict", "mixed"))
a = ap.parse_args()
base = torch.from_numpy(fe.synthetic.config_c4()).cuda().float()
eng = fe.FrontEnd(1080, 1920, a.frames, laplacian=fe.LaplacianParams(1.0, 3, 10),
                  bilateral=fe.BilateralParams(0.1, 0.15, 3, 5), src_dtype=torch.float32,
                  graph=False, precision=a.precision)
eng.src.copy_(base.expand_as(eng.src))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for k in range(a.steps):
    ev[0].record()
    eng.launch()
    ev[1].record()
    torch.cuda.synchronize()
    print(f"step {k}: {ev[0].elapsed_time(ev[1]):.3f} ms, n_tri {eng.n_tri[0].item()}")
