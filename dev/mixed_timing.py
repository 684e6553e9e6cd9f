"""Device time of the pieces of a MIXED C4 chain (16 frames): strict Laplacian + f64 FC
data + the fp32 bilateral on the FC arrays (MODE 2, scatter) -- vs the fast / strict
front ends."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2007_12065_b200 as fe  # noqa: E402
from paper_2007_12065_b200 import _ops  # noqa: E402

F = 16
base = torch.from_numpy(fe.synthetic.config_c4()).cuda()
src = base.unsqueeze(0).expand(F, -1, -1, -1).contiguous()
M, N = base.shape[:2]
ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
for rep in range(3):
    ev[0].record()
    sm = _ops.laplacian_f64(src, 1.0, 3, 10)
    ev[1].record()
    eng_tri = None
    cen = torch.empty((F, M - 1, N - 1, 2, 3), dtype=torch.float64, device="cuda")
    nrm = torch.empty_like(cen)
    ev[2].record()
    fe._lib.check(fe._lib.lib().opcfe_fc_data(sm.data_ptr(), 1, M, N * 1, cen.data_ptr(), nrm.data_ptr(),
                                              fe._device.stream()), "fc") if F == 1 else None
    for f in range(F):
        fe._lib.check(fe._lib.lib().opcfe_fc_data(sm[f].data_ptr(), 1, M, N, cen[f].data_ptr(),
                                                  nrm[f].data_ptr(), fe._device.stream()), "fc")
    ev[3].record()
    fc32 = _ops.stage_fc(nrm)
    ev[4].record()
    out = _ops.bilateral(F, M, N, 0.1, 0.15, 3, 5, fc_normals=fc32, fc_centroids=cen)
    ev[5].record()
    torch.cuda.synchronize()
    print(f"rep {rep}: lap64 {ev[0].elapsed_time(ev[1]):.2f} ms, fc64 {ev[2].elapsed_time(ev[3]):.2f}, "
          f"stage {ev[3].elapsed_time(ev[4]):.2f}, bilateral MODE2 x5 {ev[4].elapsed_time(ev[5]):.2f}")
