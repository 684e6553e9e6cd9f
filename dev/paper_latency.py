"""Single-frame device latency at the paper's sizes:
Laplacian 1 / 5 iterations and bilateral (incl. FC normals + centroids) 1 / 5 iterations on one
500x500 and one 120x212 frame: mesh alone, Laplacian + mesh, mesh + bilateral, each a CUDA-graph
replay, device time per call (single frames are launch-latency bound: ~3 us per kernel)."""
import sys, json
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_2007_12065_b200 as fe

def t(eng, reps=200):
    eng.launch(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        eng.launch()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

out = {}
for (M, N) in ((500, 500), (212, 120)):
    opc = fe.synthetic.room_scene(n=max(M, N), noise=0.002, seed=1)[:M, :N].copy()
    src = torch.from_numpy(opc).float().cuda().unsqueeze(0)
    for it in (1, 5):
        lap = fe.FrontEnd(M, N, 1, laplacian=fe.LaplacianParams(1.0, 3, it), bilateral=None,
                          normals=False, halfedges=False)
        lap.src.copy_(src)
        mesh = fe.FrontEnd(M, N, 1, laplacian=None, bilateral=None, normals=False)
        mesh.src.copy_(src)
        full = fe.FrontEnd(M, N, 1, laplacian=None, bilateral=fe.BilateralParams(0.1, 0.15, 3, it))
        full.src.copy_(src)
        tl, tm, tf = t(lap), t(mesh), t(full)
        out[f"{M}x{N} it={it}"] = {"mesh_only_ms": round(tm, 4),
                                   "laplacian_plus_mesh_ms": round(tl, 4),
                                   "mesh_plus_bilateral_ms": round(tf, 4)}
print(json.dumps(out, indent=1))
