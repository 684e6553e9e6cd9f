"""One mixed-precision Laplacian chain (C4, 16 frames, 2 passes) for ncu captures."""
import os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2007_12065_b200 as fe
eng = fe.FrontEnd(1080, 1920, 16, laplacian=fe.LaplacianParams(1.0, 3, 2), bilateral=None, src_dtype=torch.float64, graph=False, precision="mixed")
eng.src.copy_(torch.from_numpy(fe.synthetic.config_c4()).cuda().expand_as(eng.src))
eng.run(eng.src); torch.cuda.synchronize(); print("ok")
