"""Which bar a failing mixed-precision random cloud misses (dev/stress_mixed.py seeds)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import test_gpu_vs_reference as R
import paper_2007_12065_b200 as fe

ref = R.ref.__wrapped__()
for seed in [int(s) for s in sys.argv[1:]] or [156, 200]:
    rng = np.random.default_rng(9300 + seed)
    opc = R.random_cloud(rng)
    M, N = opc.shape[:2]
    lap = (float(rng.uniform(0.2, 1.0)), 3, int(rng.integers(1, 6)))
    bil = (float(rng.uniform(0.02, 0.3)), float(rng.uniform(0.05, 0.5)),
           int(rng.choice([3, 5, 7])), int(rng.integers(1, 4)))
    r_sm = ref.smoothing.laplacian_filter_opc(opc, ref.smoothing.LaplacianParams(*lap))
    r_mesh = ref.mesh.mesh_from_opc(r_sm)
    r_n = ref.smoothing.bilateral_filter_opc(r_sm, ref.smoothing.BilateralParams(*bil), r_mesh.trimap)
    out = {}
    for prec in ("mixed", "fast", "strict"):
        eng = fe.FrontEnd(M, N, 1, laplacian=fe.LaplacianParams(*lap),
                          bilateral=fe.BilateralParams(*bil), src_dtype=torch.float64,
                          precision=prec)
        res = eng.run(torch.from_numpy(opc).cuda().unsqueeze(0))
        T = res.n_tri[0]
        pts = res.points[0].cpu().numpy()
        g_n = res.normals[0, :T].cpu().numpy().astype(np.float64)
        bad = np.isnan(r_n).any(1)
        gbad = np.isnan(g_n).any(1)
        info = dict(pts_same=R.same(pts.astype(np.float64), r_sm) if prec != "fast" else None,
                    trimap=np.array_equal(res.trimap[0].cpu().numpy(), r_mesh.trimap),
                    tris=T == len(r_mesh.triangles) and
                    np.array_equal(res.triangles[0, :T].cpu().numpy(), r_mesh.triangles),
                    nan_same=np.array_equal(gbad, bad) if len(gbad) == len(bad) else 'len')
        if len(gbad) == len(bad):
            ok = ~bad & ~gbad
            e = np.linalg.norm(g_n[ok] - r_n[ok], axis=1)
            info['err'] = float(e.max()) if len(e) else 0.0
            if info['nan_same'] is not True:
                d = np.nonzero(gbad != bad)[0][:5]
                info['nan_diff'] = [(int(i), r_n[i].tolist(), g_n[i].tolist()) for i in d]
        out[prec] = info
    print(seed, (M, N), lap, bil)
    for k, v in out.items():
        print('  ', k, v)
