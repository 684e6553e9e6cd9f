"""GPU parity: the CUDA path (through the C ABI) against the oracle and the golden vectors.

Bars (north-star + SURVEY.md 8c precision contract):
  * triangles / trimap / halfedges / validity / l_max flags: bit-exact;
  * fp64 drop-in normals & FC data (compute_normals, compute_fc_triangle_data): bit-exact;
  * Laplacian vertices: per vertex |g - r| <= 1e-5 * max(|r|, rms|r|) (norm-wise
    relative); unchanged vertices (ring, NaN, isolated) bit-identical;
  * bilateral normals (unit vectors): per triangle |g - r| <= 1e-5; NaN masks equal.
Drop-in calls run with precision "fast" here (module fixture).
Fused fp32 pipeline: per-stage parity on identical inputs -- each oracle stage consumes
the GPU's fp32 intermediate (upcast to f64) -- plus end-to-end bit-exact topology.
"""

import os

import numpy as np
import pytest
import torch

from conftest import grid_opc, load_golden
from oracle import c_oracle
from oracle import flatpoly_oracle as fo

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

TOL = 1e-5


@pytest.fixture(scope="module")
def fe():
    import paper_2007_12065_b200 as m
    return m


@pytest.fixture(autouse=True, scope="module")
def _fast_precision():
    """This module checks the fp32 ("fast") drop-in path against the 1e-5 contract; the
    strict fp64 path (the float64 default) is checked in test_gpu_strict.py."""
    from paper_2007_12065_b200 import smoothing
    old = smoothing.get_precision()
    smoothing.set_precision("fast")
    yield
    smoothing.set_precision(old)


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(np.isnan(a), np.isnan(b)) and \
        np.array_equal(np.nan_to_num(a), np.nan_to_num(b))


def teq(a, b):
    """bit-equal device tensors, NaN == NaN"""
    a, b = a.contiguous(), b.contiguous()
    if a.is_floating_point():
        return torch.equal(torch.isnan(a), torch.isnan(b)) and \
            torch.equal(torch.nan_to_num(a), torch.nan_to_num(b))
    return torch.equal(a, b)


def assert_vertices_close(g, r, tol=TOL):
    g = np.asarray(g, dtype=np.float64).reshape(-1, 3)
    r = np.asarray(r, dtype=np.float64).reshape(-1, 3)
    assert np.array_equal(np.isnan(g), np.isnan(r))
    ok = np.isfinite(r).all(axis=1)
    if not ok.any():
        return
    err = np.linalg.norm(g[ok] - r[ok], axis=1)
    mag = np.linalg.norm(r[ok], axis=1)
    scale = np.maximum(mag, np.sqrt(np.mean(mag ** 2)))
    worst = float(np.max(err / scale))
    assert worst <= tol, f"norm-wise relative error {worst:.3e} > {tol}"


def assert_normals_close(g, r, tol=TOL):
    g = np.asarray(g, dtype=np.float64).reshape(-1, 3)
    r = np.asarray(r, dtype=np.float64).reshape(-1, 3)
    assert g.shape == r.shape
    assert np.array_equal(np.isnan(g).any(axis=1), np.isnan(r).any(axis=1))
    ok = ~np.isnan(r).any(axis=1)
    if ok.any():
        worst = float(np.max(np.linalg.norm(g[ok] - r[ok], axis=1)))
        assert worst <= tol, f"normal error {worst:.3e} > {tol}"


def check_twins(tris, he):
    """Reference acceptance #05 properties: involution + reversed vertex pairs."""
    tris = np.asarray(tris)
    he = np.asarray(he)
    assert len(he) == 3 * len(tris)
    e = np.nonzero(he >= 0)[0]
    assert np.all(he[he[e]] == e)
    flat = tris.ravel()
    t, k = np.divmod(e, 3)
    tw = he[e]
    tt, tk = np.divmod(tw, 3)
    assert np.all(flat[tw] == flat[3 * t + (k + 1) % 3])
    assert np.all(flat[3 * tt + (tk + 1) % 3] == flat[e])


# --------------------------------------------------------------- golden: topology
TOPO = load_golden("topology")


@pytest.mark.parametrize("case", sorted(TOPO))
def test_golden_topology(fe, case):
    g = TOPO[case]
    opc = g["opc"]
    M, N = opc.shape[:2]
    tris, trimap = fe.extract_triangles_opc(opc)
    assert tris.dtype == np.int64 and trimap.dtype == np.int64
    assert np.array_equal(tris, g["triangles"])
    assert np.array_equal(trimap, g["trimap"])
    assert np.array_equal(fe.extract_halfedges_opc(trimap, M, N), g["halfedges"])
    mesh = fe.mesh_from_opc(opc)
    assert np.array_equal(mesh.triangles, g["triangles"])
    assert np.array_equal(mesh.halfedges, g["halfedges"])
    assert np.array_equal(mesh.trimap, g["trimap"])
    assert same(mesh.normals, g["normals"])                   # fp64 bit-exact
    assert np.shares_memory(mesh.points, opc) and mesh.grid_shape == (M, N)
    cen, nrm = fe.compute_fc_triangle_data(opc)
    assert same(cen, g["fc_centroids"]) and same(nrm, g["fc_normals"])


def test_known_answers(fe):
    tris, trimap = fe.extract_triangles_opc(grid_opc(2, 2))
    assert tris.tolist() == [[3, 1, 0], [0, 2, 3]] and trimap.tolist() == [0, 1]
    o = grid_opc(2, 2)
    o[0, 1] = np.nan
    tris, trimap = fe.extract_triangles_opc(o)
    assert tris.tolist() == [[0, 2, 3]] and trimap.tolist() == [-1, 0]
    _, trimap = fe.extract_triangles_opc(grid_opc(2, 2))
    assert fe.extract_halfedges_opc(trimap, 2, 2).tolist() == [-1, -1, 5, -1, -1, 2]
    with pytest.raises(fe.DegenerateInputError):
        fe.extract_triangles_opc(grid_opc(1, 5))


def test_acceptance05_random_grids(fe):
    """500 random OPCs 2..50^2, NaN 0-50 %: bit-exact vs the oracle + twin properties."""
    rng = np.random.default_rng(11)
    for _ in range(500):
        M = int(rng.integers(2, 51))
        N = int(rng.integers(2, 51))
        opc = grid_opc(M, N)
        opc[..., 2] = rng.normal(0, 0.1, (M, N))
        opc[rng.random((M, N)) < rng.uniform(0.0, 0.5)] = np.nan
        mesh = fe.mesh_from_opc(opc)
        tris, trimap, he = c_oracle.triangulate(opc)
        assert np.array_equal(mesh.triangles, tris)
        assert np.array_equal(mesh.trimap, trimap)
        assert np.array_equal(mesh.halfedges, he)
        check_twins(mesh.triangles, mesh.halfedges)


# (3, 4099) / (5, 12003): rows of more than one 4096-quad scan segment of the row CTA
# (triangulate.cu: carries between segments); (9000, 3): many 2-quad rows
@pytest.mark.parametrize("shape", [(2, 1000), (1000, 2), (3, 3), (97, 33), (64, 1024),
                                   (300, 257), (1080, 1920), (3, 4099), (5, 12003),
                                   (9000, 3)])
def test_topology_shapes(fe, shape):
    M, N = shape
    rng = np.random.default_rng(M * 7 + N)
    opc = grid_opc(M, N)
    opc[..., 2] = rng.normal(0, 0.01, (M, N))
    opc[rng.random((M, N)) < 0.1] = np.nan
    mesh = fe.mesh_from_opc(opc)
    tris, trimap, he = c_oracle.triangulate(opc)
    assert np.array_equal(mesh.triangles, tris)
    assert np.array_equal(mesh.trimap, trimap)
    assert np.array_equal(mesh.halfedges, he)
    assert same(mesh.normals, c_oracle.triangle_normals(opc, tris))


def test_all_nan_and_degenerate(fe):
    mesh = fe.mesh_from_opc(np.full((6, 6, 3), np.nan))
    assert mesh.num_triangles == 0 and len(mesh.halfedges) == 0
    assert np.all(mesh.trimap == -1)
    mesh = fe.mesh_from_opc(np.zeros((5, 5, 3)))        # coincident points
    assert mesh.num_triangles == 32 and np.all(np.isnan(mesh.normals))


# --------------------------------------------------------------- golden: Laplacian
LAP = load_golden("laplacian")


@pytest.mark.parametrize("case", sorted(LAP))
def test_golden_laplacian(fe, case):
    g = LAP[case]
    lam, k, it = g["params"]
    out = fe.laplacian_filter_opc(g["opc"], fe.LaplacianParams(lam=lam, kernel_size=int(k),
                                                               iterations=int(it)))
    assert out.dtype == np.float64 and out.shape == g["opc"].shape
    assert_vertices_close(out, g["out"])
    # outer ring and non-finite vertices come back bit-identical (test_smoothing.py:45-57)
    for sl in (np.s_[0], np.s_[-1], np.s_[:, 0], np.s_[:, -1]):
        assert same(out[sl], g["opc"][sl])
    bad = ~np.isfinite(g["opc"]).all(axis=2)
    assert same(out[bad], g["opc"][bad])
    out2 = fe._kernels.laplacian_filter(g["opc"], lam, int(k), int(it))
    assert same(out2, out)


def test_laplacian_hand_rolled_update(fe):
    opc = fe.synthetic.flat_plane_opc(7, 7, spacing=1.0)
    opc[3, 3, 2] = 0.5
    out = fe.laplacian_filter_opc(opc, fe.LaplacianParams(lam=1.0, kernel_size=3, iterations=1))
    v = opc[3, 3]
    d = opc[2:5, 2:5].reshape(-1, 3) - v
    d = np.delete(d, 4, axis=0)
    w = 1.0 / np.linalg.norm(d, axis=1)
    expected = v + (w[:, None] * d).sum(0) / w.sum()
    assert np.max(np.abs(out[3, 3] - expected)) < 1e-6
    assert out[3, 3, 2] < opc[3, 3, 2]


def test_laplacian_kernel5_two_ring_and_fixed_point(fe):
    opc = fe.synthetic.flat_plane_opc(11, 11, spacing=1.0)
    opc[3, 3, 2] = 1.0
    out3 = fe.laplacian_filter_opc(opc, fe.LaplacianParams(kernel_size=3))
    out5 = fe.laplacian_filter_opc(opc, fe.LaplacianParams(kernel_size=5))
    assert out3[5, 5, 2] == 0.0 and out5[5, 5, 2] > 0.0
    flat = fe.synthetic.flat_plane_opc(10, 12, spacing=0.1)
    out = fe.laplacian_filter_opc(flat, fe.LaplacianParams(lam=1.0, kernel_size=3, iterations=3))
    assert np.max(np.abs(out - flat)) < 1e-6


@pytest.mark.parametrize("k,it", [(3, 1), (3, 4), (5, 2), (7, 1), (9, 2), (17, 1)])
@pytest.mark.parametrize("shape", [(41, 37), (96, 130), (17, 250)])
def test_laplacian_vs_oracle(fe, k, it, shape):
    M, N = shape
    rng = np.random.default_rng(k * 100 + it)
    opc = fe.synthetic.flat_plane_opc(M, N, spacing=0.01, noise=0.002, seed=k + it)
    opc[rng.random((M, N)) < 0.07] = np.nan
    if min(M, N) < k:
        return
    out = fe.laplacian_filter_opc(opc, fe.LaplacianParams(lam=0.9, kernel_size=k, iterations=it))
    assert_vertices_close(out, c_oracle.laplacian_filter(opc, 0.9, k, it))


def test_laplacian_grid_smaller_than_kernel(fe):
    with pytest.raises(fe.DegenerateInputError, match="smaller than the filter kernel"):
        fe.laplacian_filter_opc(np.zeros((2, 9, 3)), fe.LaplacianParams(kernel_size=3))


def test_laplacian_torch_tensor_stays_on_device(fe):
    opc = torch.from_numpy(fe.synthetic.flat_plane_opc(20, 24, noise=0.01, seed=2)).float().cuda()
    out = fe.laplacian_filter_opc(opc, fe.LaplacianParams(iterations=2))
    assert isinstance(out, torch.Tensor) and out.is_cuda and out.dtype == torch.float32
    ref = c_oracle.laplacian_filter(opc.double().cpu().numpy(), 1.0, 3, 2)
    assert_vertices_close(out.cpu().numpy(), ref)


# --------------------------------------------------------------- golden: bilateral
BIL = load_golden("bilateral")


@pytest.mark.parametrize("case", sorted(c for c in BIL if c.startswith("iter")))
def test_golden_bilateral_iterate(fe, case):
    g = BIL[case]
    sl, sa, k, it = g["params"]
    out = fe._kernels.bilateral_iterate(g["centroids"], g["normals"], sl, sa, int(k), int(it))
    assert out.shape == g["normals"].shape and out.dtype == np.float64
    assert_normals_close(out, g["out"])
    assert_normals_close(out, g["out_native"])


@pytest.mark.parametrize("case", sorted(c for c in BIL if not c.startswith("iter")))
def test_golden_bilateral_filter_opc(fe, case):
    g = BIL[case]
    sl, sa, k, it = g["params"]
    out = fe.bilateral_filter_opc(g["opc"], fe.BilateralParams(sl, sa, int(k), int(it)))
    assert out.dtype == np.float64
    assert_normals_close(out, g["out"])
    norms = np.linalg.norm(out[np.isfinite(out).all(1)], axis=1)
    assert np.allclose(norms, 1.0, atol=1e-6)


def test_bilateral_right_angle_edge_preserved(fe):
    g = BIL["rightangle"]
    out = fe.bilateral_filter_opc(g["opc"], fe.BilateralParams(sigma_length=1.0, sigma_angle=0.1))
    tris, _ = fe.extract_triangles_opc(g["opc"])
    cents = g["opc"].reshape(-1, 3)[tris].mean(axis=1)
    flat_side = (cents[:, 2] > -1e-9) & (cents[:, 0] < 0.2)
    wall_side = cents[:, 2] < -0.05
    ang_f = np.degrees(np.arccos(np.clip(out[flat_side] @ [0, 0, 1.0], -1, 1)))
    ang_w = np.degrees(np.arccos(np.clip(out[wall_side] @ [1.0, 0, 0], -1, 1)))
    assert ang_f.max() < 2.0 and ang_w.max() < 2.0


@pytest.mark.parametrize("k,it", [(3, 1), (3, 3), (5, 2), (7, 1), (9, 1)])
def test_bilateral_vs_oracle(fe, k, it):
    rng = np.random.default_rng(k + 10 * it)
    opc = fe.synthetic.room_scene(n=70, noise=0.002, seed=k)
    opc[rng.random(opc.shape[:2]) < 0.05] = np.nan
    out = fe.bilateral_filter_opc(opc, fe.BilateralParams(0.1, 0.15, k, it))
    ref = c_oracle.front_end(opc, None, (0.1, 0.15, k, it))["normals"]
    assert_normals_close(out, ref)


def test_bilateral_given_trimap_and_small_grid(fe):
    opc = np.full((2, 2, 3), np.nan)
    opc[0, 0], opc[0, 1], opc[1, 1] = [0, 0, 0], [1, 0, 0], [1, -1, 0]
    out = fe.bilateral_filter_opc(opc, fe.BilateralParams())
    assert out.shape == (1, 3) and np.allclose(out[0], [0, 0, 1.0], atol=1e-12)
    opc = fe.synthetic.flat_plane_opc(6, 6, spacing=0.1)
    _, trimap = fe.extract_triangles_opc(opc)
    out = fe.bilateral_filter_opc(opc, fe.BilateralParams(iterations=3), trimap)
    assert np.allclose(out, np.tile([0, 0, 1.0], (len(out), 1)), atol=1e-7)


# --------------------------------------------------------------- fused pipeline
FE = load_golden("frontend")


def _engine_run(fe, opc, lap, bil, l_max=None, frames=1, dtype=torch.float32, graph=True):
    M, N = opc.shape[-3:-1]
    eng = fe.FrontEnd(M, N, frames, laplacian=lap, bilateral=bil, l_max=l_max,
                      src_dtype=dtype, graph=graph)
    src = torch.from_numpy(np.ascontiguousarray(opc)).to("cuda", dtype).reshape(frames, M, N, 3)
    res = eng.run(src)
    torch.cuda.synchronize()
    return eng, res


def _bilateral_per_iteration(res, bil, sm_gpu, trimap, T):
    """Bilateral parity per iteration (each iteration is one kernel launch, i.e. one
    _kernels.bilateral_iterate(.., iterations=1) call of the reference): every launch is
    within 1e-5 of one oracle iteration applied to the same input normals (the GPU's
    previous fp32 output, upcast), and the fused B-iteration output equals the chain
    of single-iteration launches bit for bit.  The chained B-iteration error against
    the fp64 chain is returned as information (fp32 rounding compounds over iterations
    at a few bistable triangles)."""
    from paper_2007_12065_b200 import _ops
    M, N = sm_gpu.shape[:2]
    Mq, Nq = M - 1, N - 1
    grid, _ = _ops.stage_in(res.points[0].contiguous(), want_points=True, want_mask=False)
    cen, ref_in = c_oracle.compute_fc_triangle_data(sm_gpu)
    tm = res.trimap[:1].contiguous()
    prev = None
    args = (bil.sigma_length, bil.sigma_angle, bil.kernel_size, 1)
    for it in range(1, bil.iterations + 1):
        ref = c_oracle.bilateral_iterate(cen, ref_in, *args)
        if it < bil.iterations:
            out = _ops.bilateral(1, M, N, *args, grid=grid, fc_normals=prev)
            g = out[0, :, :6 * Nq].reshape(Mq, Nq, 2, 3).cpu().numpy().astype(np.float64)
            assert_normals_close(g, ref)
            ref_in, prev = g, out
        else:
            out = _ops.bilateral(1, M, N, *args, grid=grid, fc_normals=prev, trimap=tm,
                                 out_rows=T)[0]
            assert_normals_close(out.cpu().numpy(), c_oracle.gather(ref, trimap, T))
            assert teq(out, res.normals[0, :T])
    full = c_oracle.bilateral_iterate(cen, c_oracle.compute_fc_triangle_data(sm_gpu)[1],
                                      bil.sigma_length, bil.sigma_angle, bil.kernel_size,
                                      bil.iterations)
    err = np.linalg.norm(res.normals[0, :T].cpu().numpy() - c_oracle.gather(full, trimap, T),
                         axis=1)
    err = err[np.isfinite(err)]
    assert err.max() < 1e-3
    return float(err.max()), int((err > TOL).sum())


def _per_stage_check(fe, opc, lap, bil, l_max=None, res=None):
    """Per-stage parity of one frame: each oracle stage consumes the GPU's fp32 output."""
    x32 = np.asarray(opc, dtype=np.float32).astype(np.float64)
    sm_gpu = res.points.cpu().numpy()[0].astype(np.float64)
    if lap is not None:
        # per pass: every GPU pass within 1e-5 of one fp64 reference pass on the same input
        # (chained fp32 vs chained fp64 is ill-conditioned where the 1/|d| weights collapse
        # two vertices onto each other), and the fused L-pass result equals the chain of
        # single passes bit for bit
        cur = np.asarray(opc, dtype=np.float32)
        one = fe.LaplacianParams(lap.lam, lap.kernel_size, 1)
        for _ in range(lap.iterations):
            g = np.asarray(fe.laplacian_filter_opc(cur, one), dtype=np.float32)
            assert_vertices_close(g, c_oracle.laplacian_filter(cur.astype(np.float64), lap.lam,
                                                               lap.kernel_size, 1))
            cur = g
        assert same(res.points.cpu().numpy()[0], cur)
    else:
        assert same(sm_gpu, x32)
    T = res.n_tri[0]
    tris, trimap, he = c_oracle.triangulate(sm_gpu)
    assert T == len(tris)
    assert np.array_equal(res.triangles[0, :T].cpu().numpy(), tris)
    assert np.array_equal(res.trimap[0].cpu().numpy(), trimap)
    assert np.array_equal(res.halfedges[0, :3 * T].cpu().numpy(), he)
    normals = res.normals[0, :T].cpu().numpy()
    if bil is not None:
        _bilateral_per_iteration(res, bil, sm_gpu, trimap, T)
    else:
        # fp64 math on the fp32 grid -> exactly float32(oracle)
        ref = c_oracle.triangle_normals(sm_gpu, tris).astype(np.float32)
        assert same(normals, ref)
    if l_max is not None:
        m = res.lmax_mask[0, :T].cpu().numpy().astype(bool)
        assert np.array_equal(m, c_oracle.max_edge_mask(sm_gpu, tris, l_max))
    # topology is invariant under the Laplacian: vs the raw input
    t0, tm0, _ = c_oracle.triangulate(np.asarray(opc, dtype=np.float64))
    assert np.array_equal(tm0, trimap)


def test_front_end_room_golden(fe):
    g = FE["room"]
    lap = fe.LaplacianParams(*[float(g["lap"][0]), int(g["lap"][1]), int(g["lap"][2])])
    bil = fe.BilateralParams(float(g["bil"][0]), float(g["bil"][1]), int(g["bil"][2]),
                             int(g["bil"][3]))
    _, res = _engine_run(fe, g["opc"], lap, bil, l_max=0.05)
    _per_stage_check(fe, g["opc"], lap, bil, 0.05, res)
    T = res.n_tri[0]
    assert np.array_equal(res.triangles[0, :T].cpu().numpy(), g["triangles"])
    assert np.array_equal(res.halfedges[0, :3 * T].cpu().numpy(), g["halfedges"])
    # information only: the chained fp32 result against the fp64 chain
    chained = np.linalg.norm(res.normals[0, :T].cpu().numpy() - g["normals"], axis=1)
    assert np.nanmax(chained) < 1e-2


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4"])
def test_front_end_configs(fe, cfg):
    syn = fe.synthetic
    lap = bil = None
    l_max = None
    if cfg == "C1":
        opc = syn.config_c1()
        lap, bil = fe.LaplacianParams(1.0, 3, 1), fe.BilateralParams(0.1, 0.15, 3, 1)
    elif cfg == "C2":
        opc = syn.config_c2()
        lap, bil = fe.LaplacianParams(1.0, 3, 3), fe.BilateralParams(0.1, 0.15, 3, 2)
    elif cfg == "C3":
        opc = syn.config_c3()
        lap, l_max = fe.LaplacianParams(1.0, 3, 5), 0.5
    else:
        opc = syn.config_c4()
        lap, bil = fe.LaplacianParams(1.0, 3, 10), fe.BilateralParams(0.1, 0.15, 3, 5)
    _, res = _engine_run(fe, opc, lap, bil, l_max)
    _per_stage_check(fe, opc, lap, bil, l_max, res)
    T = res.n_tri[0]
    check_twins(res.triangles[0, :T].cpu().numpy(), res.halfedges[0, :3 * T].cpu().numpy())


def test_front_end_batch_equals_single(fe):
    frames = fe.synthetic.config_c5_frames(3)[:, :120, :200]
    lap, bil = fe.LaplacianParams(1.0, 3, 3), fe.BilateralParams(0.1, 0.15, 3, 2)
    _, res = _engine_run(fe, frames, lap, bil, l_max=0.01, frames=3)
    for f in range(3):
        _, r1 = _engine_run(fe, frames[f], lap, bil, l_max=0.01)
        T = r1.n_tri[0]
        assert res.n_tri[f] == T
        assert teq(res.points[f], r1.points[0])
        assert torch.equal(res.triangles[f, :T], r1.triangles[0, :T])
        assert torch.equal(res.halfedges[f, :3 * T], r1.halfedges[0, :3 * T])
        assert teq(res.normals[f, :T], r1.normals[0, :T])
        assert torch.equal(res.lmax_mask[f, :T], r1.lmax_mask[0, :T])


def test_front_end_f64_source_and_no_graph(fe):
    opc = fe.synthetic.config_c2()[:100, :130]
    lap, bil = fe.LaplacianParams(0.7, 5, 2), fe.BilateralParams(0.1, 0.15, 3, 3)
    _, r64 = _engine_run(fe, opc, lap, bil, dtype=torch.float64, graph=False)
    _, r32 = _engine_run(fe, opc, lap, bil, dtype=torch.float32, graph=True)
    assert teq(r64.points, r32.points)
    T = r64.n_tri[0]
    assert T == r32.n_tri[0]
    assert teq(r64.normals[:, :T], r32.normals[:, :T])
    assert teq(r64.triangles[:, :T], r32.triangles[:, :T])
    _per_stage_check(fe, opc, lap, bil, None, r64)


def test_front_end_function_numpy(fe):
    g = FE["lidar"]
    sm, mesh, mask = fe.front_end(g["opc"], fe.LaplacianParams(1.0, 3, 5), None, l_max=0.5)
    assert np.array_equal(mesh.triangles, g["triangles"])
    assert np.array_equal(mesh.halfedges, g["halfedges"])
    assert_vertices_close(sm, g["smoothed"])
    keep = g["labels_lmaxinf"] != 255
    assert np.array_equal(mask[keep], g["labels_lmax0.5"][keep] == 255)


def test_lmax_mask_golden(fe):
    g = FE["room"]
    mesh = fe.HalfEdgeMesh(points=g["smoothed"].reshape(-1, 3), triangles=g["triangles"],
                           halfedges=g["halfedges"])
    keep = g["labels_lmaxinf"] != 255
    for l_max in (0.05, 0.5):
        m = fe.max_edge_mask(mesh, l_max)
        assert np.array_equal(m[keep], g[f"labels_lmax{l_max}"][keep] == 255)
    g = FE["grid3"]
    mesh = fe.mesh_from_opc(g["opc"])
    assert np.all(fe.max_edge_mask(mesh, 0.5)) and not np.any(fe.max_edge_mask(mesh, 2.0))


def _np_lmax(pts, tris, l_max):
    """segmentation.py:59-67,73: np.maximum of the three np.linalg.norm edge lengths > l_max"""
    a, b, c = pts[tris[:, 0]], pts[tris[:, 1]], pts[tris[:, 2]]
    e = np.maximum(np.linalg.norm(b - a, axis=1),
                   np.maximum(np.linalg.norm(c - b, axis=1), np.linalg.norm(a - c, axis=1)))
    with np.errstate(invalid="ignore"):
        return e > l_max


def test_lmax_threshold_at_exact_edge_lengths(fe):
    """The kernels compare squared lengths against sq_threshold(l_max) (no sqrt): l_max
    set to an exact edge length, one ulp either side, 0, negative, inf, NaN vertices."""
    rng = np.random.default_rng(77)
    pts = rng.normal(scale=0.3, size=(400, 3))
    pts[5] = np.nan
    tris = rng.integers(0, 400, size=(2000, 3))
    tris[:40, 1] = tris[:40, 0]                       # zero-length edges
    mesh = fe.HalfEdgeMesh(points=pts, triangles=tris, halfedges=None)
    lens = np.linalg.norm(pts[tris[:, 1]] - pts[tris[:, 0]], axis=1)
    cands = [0.0, -1.0, np.inf, 1e-300, 1e300]
    for L in lens[np.isfinite(lens)][:60]:
        cands += [L, np.nextafter(L, 0), np.nextafter(L, np.inf)]
    for l_max in cands:
        assert np.array_equal(fe.max_edge_mask(mesh, l_max), _np_lmax(pts, tris, l_max)), l_max
    # the fused fp32 front end: l_max = exact edge lengths of the fp32 grid
    opc = grid_opc(24, 31) * 0.05 + rng.normal(scale=0.02, size=(24, 31, 3))
    opc[rng.random((24, 31)) < 0.1] = np.nan
    opc = opc.astype(np.float32)
    for k in range(4):
        sm = opc.astype(np.float64)
        tris_r, _, _ = c_oracle.triangulate(sm)
        p = sm.reshape(-1, 3)
        L = float(np.linalg.norm(p[tris_r[7 * k, 1]] - p[tris_r[7 * k, 0]]))
        for l_max in (L, np.nextafter(L, 0), np.nextafter(L, np.inf)):
            _, res = _engine_run(fe, opc, None, None, l_max=l_max)
            T = res.n_tri[0]
            assert np.array_equal(res.lmax_mask[0, :T].cpu().numpy().astype(bool),
                                  _np_lmax(p, tris_r, l_max)), (k, l_max)


def test_compute_normals_any_mesh(fe):
    rng = np.random.default_rng(12345)
    pts = rng.normal(size=(30, 3))
    tris = rng.integers(0, 30, size=(40, 3))
    mesh = fe.HalfEdgeMesh(points=pts, triangles=tris, halfedges=None)
    assert same(fe.compute_normals(mesh), fo.triangle_normals(pts, tris))


def test_bilateral_input_modes(fe):
    """All three kernel input modes meet the contract: FC arrays (bilateral_filter_opc),
    and the fused pipeline's point-grid first iteration + FC-normal resume iterations."""
    for seed, k, it in ((5, 3, 1), (6, 3, 3), (7, 5, 2)):
        opc = fe.synthetic.room_scene(n=97, noise=0.002, seed=seed)
        opc[np.random.default_rng(seed).random(opc.shape[:2]) < 0.05] = np.nan
        bil = (0.1, 0.15, k, it)
        # FC-array mode (fp64 FC data from the fp64 grid, like the reference)
        ref = c_oracle.front_end(opc, None, bil)["normals"]
        out = fe.bilateral_filter_opc(opc, fe.BilateralParams(*bil))
        # point-grid modes: the fused pipeline works on the fp32 grid -> per-stage input
        opc32 = opc.astype(np.float32).astype(np.float64)
        ref32 = c_oracle.front_end(opc32, None, bil)["normals"]
        _, mesh, _ = fe.front_end(opc32, None, fe.BilateralParams(*bil))
        for o, r in ((out, ref), (mesh.normals, ref32)):
            ok = np.isfinite(r).all(1)
            assert np.array_equal(ok, np.isfinite(o).all(1))
            assert_normals_close(o[ok], r[ok])


GROUPS = load_golden("groups")


@pytest.mark.parametrize("case", sorted(GROUPS))
def test_golden_group_assignment(fe, case):
    """segmentation.group_assignment drop-in: bit-exact labels (fp64 scores in the BLAS
    FMA order, fp64 edge lengths)."""
    g = GROUPS[case]
    l_max, ang = g["params"]
    mesh = fe.HalfEdgeMesh(points=g["points"], triangles=g["triangles"], halfedges=None,
                           normals=g["normals"])
    lab = fe.group_assignment(mesh, g["dominant"], l_max, ang)
    assert lab.dtype == np.uint8 and np.array_equal(lab, g["labels"])
    with pytest.raises(ValueError, match="dominant normals"):
        fe.group_assignment(mesh, np.zeros((255, 3)), l_max, ang)


def test_front_end_fused_labels(fe):
    """Labels fused after the bilateral pass == oracle group_assignment on the GPU's own
    fp32 normals / smoothed grid (per-stage parity)."""
    opc = fe.synthetic.config_c2()
    lap, bil = fe.LaplacianParams(1.0, 3, 3), fe.BilateralParams(0.1, 0.15, 3, 2)
    dn = np.array([[0, 0, 1.0], [-1.0, 0, 0], [1.0, 0, 0], [0, -1.0, 0], [0, 1.0, 0]])
    M, N = opc.shape[:2]
    eng = fe.FrontEnd(M, N, 1, laplacian=lap, bilateral=bil, l_max=0.05, dominant_normals=dn,
                      ang_min=0.96)
    res = eng.run(torch.from_numpy(opc).float().cuda().unsqueeze(0))
    torch.cuda.synchronize()
    T = res.n_tri[0]
    sm = res.points[0].cpu().numpy().astype(np.float64)
    ref = c_oracle.group_assignment(sm.reshape(-1, 3), res.triangles[0, :T].cpu().numpy(),
                                    res.normals[0, :T].cpu().numpy().astype(np.float64), dn,
                                    0.05, 0.96)
    lab = res.labels[0, :T].cpu().numpy()
    assert np.array_equal(lab, ref)
    # laplacian 3 + triangulate (count, scan, emit) 3 + l_max flags 1 + bilateral 2 + labels 1
    assert 0 < (lab == 255).sum() < T and eng.kernel_launches == 3 + 3 + 1 + 2 + 1


FASTGA = load_golden("fastga")


@pytest.mark.parametrize("case", sorted(FASTGA))
def test_golden_find_cells_and_integrate(fe, case):
    """FastGA cell search (the reference's _kernels.find_cells) and histogram votes.
    Reference bar (tests/test_kernels.py:19-33): >= 0.9999 agreement with every
    disagreement inside the 1-ring (CUDA vs glibc atan ulps); measured: exact."""
    from types import SimpleNamespace
    g = FASTGA[case]
    slope, icpt, wlo, whi = g["model"]
    cells = fe._kernels.find_cells(g["queries"], g["ids"], g["cell_normals"], g["neighbors"],
                                   slope, icpt, int(wlo), int(whi))
    assert cells.dtype == np.int64 and cells.shape == g["cells"].shape
    agree = cells == g["cells"]
    assert agree.mean() >= 0.9999
    for i in np.nonzero(~agree)[0]:
        assert cells[i] in g["neighbors"][g["cells"][i]]
    ga = SimpleNamespace(s2ids=g["ids"], normals=g["cell_normals"], neighbors=g["neighbors"],
                         model_slope=slope, model_intercept=icpt, window_lo=int(wlo),
                         window_hi=int(whi), counts=np.zeros(len(g["ids"]), dtype=np.int64))
    counts = fe.integrate_normals(ga, g["mesh_normals"], sample_pct=0.12)
    assert counts.sum() == g["counts"].sum()
    assert np.abs(counts - g["counts"]).sum() <= 2 * (~agree).sum() + 2
    assert np.array_equal(fe.find_cell_indices(ga, g["queries"][:500]), cells[:500])
    with pytest.raises(ValueError):
        fe.find_cell_indices(ga, np.zeros((2, 3)))


def test_find_cells_large_vs_c_oracle(fe):
    g = FASTGA["level4"]
    slope, icpt, wlo, whi = g["model"]
    rng = np.random.default_rng(3)
    q = rng.normal(size=(400000, 3))
    ref = c_oracle.find_cells(q, g["ids"], g["cell_normals"], g["neighbors"], slope, icpt,
                              int(wlo), int(whi))
    got = fe._kernels.find_cells(q, g["ids"], g["cell_normals"], g["neighbors"], slope, icpt,
                                 int(wlo), int(whi))
    agree = got == ref
    assert agree.mean() >= 0.9999
    for i in np.nonzero(~agree)[0]:
        assert got[i] in g["neighbors"][ref[i]]


@pytest.mark.parametrize("per_slot", [None, 1, 2])
def test_host_pipeline_matches_device_engine(fe, per_slot):
    """HostPipeline (overlapped H2D / graph / D2H per chunk of frames) returns exactly what
    the device engine computes, with D2H sized by each frame's triangle count -- one frame
    per slot, two (a partial last chunk), and the default (all five in one slot)."""
    frames = fe.synthetic.config_c5_frames(5)[:, :90, :130]
    lap, bil = fe.LaplacianParams(1.0, 3, 2), fe.BilateralParams(0.1, 0.15, 3, 2)
    pipe = fe.HostPipeline(90, 130, laplacian=lap, bilateral=bil, frames_per_slot=per_slot)
    host = torch.from_numpy(frames).pin_memory()
    res = pipe.run(host)
    res = pipe.run(host)                                 # reuse: slots and buffers recycled
    torch.cuda.synchronize()
    _, ref = _engine_run(fe, frames, lap, bil, frames=5, dtype=torch.float64)
    for f in range(5):
        T = ref.n_tri[f]
        assert res.n_tri[f] == T
        assert teq(res.points[f], ref.points[f].cpu())
        assert teq(res.trimap[f], ref.trimap[f].cpu())
        assert teq(res.triangles[f, :T], ref.triangles[f, :T].cpu())
        assert teq(res.halfedges[f, :3 * T], ref.halfedges[f, :3 * T].cpu())
        assert teq(res.normals[f, :T], ref.normals[f, :T].cpu())
    assert pipe.h2d_bytes == host.numel() * 8 and pipe.d2h_bytes > 0



def test_frames_from_files_through_host_pipeline(fe, tmp_path):
    """OPC ingestion -> front end: grid-text and binary-PLY frame files read by the native
    loader into pinned batches (FrameFileReader) give exactly the device engine's result
    on the in-memory frames (the loader is bit-exact, so the whole path is)."""
    from paper_2007_12065_b200 import io as fio
    frames = fe.synthetic.config_c5_frames(4)[:, :70, :110]
    M, N = frames.shape[1:3]
    paths = []
    for f in range(4):
        if f % 2:
            paths.append(tmp_path / f"f{f}.ply")
            fio.write_ply(paths[-1], frames[f].reshape(-1, 3), binary=True, grid=(M, N))
        else:
            paths.append(tmp_path / f"f{f}.grid")
            with open(paths[-1], "w") as fh:
                fh.write(f"{M} {N}\n")
                np.savetxt(fh, frames[f].reshape(-1, 3), fmt="%.17g")
    lap, bil = fe.LaplacianParams(1.0, 3, 2), fe.BilateralParams(0.1, 0.15, 3, 2)
    pipe = fe.HostPipeline(M, N, laplacian=lap, bilateral=bil)
    _, ref = _engine_run(fe, frames, lap, bil, frames=4, dtype=torch.float64)
    f0 = 0
    for batch in fio.FrameFileReader(paths, batch=3):
        assert batch.is_pinned()
        res = pipe.run(batch)
        torch.cuda.synchronize()
        for j in range(batch.shape[0]):
            f = f0 + j
            T = ref.n_tri[f]
            assert res.n_tri[j] == T
            assert teq(res.points[j], ref.points[f].cpu())
            assert teq(res.triangles[j, :T], ref.triangles[f, :T].cpu())
            assert teq(res.halfedges[j, :3 * T], ref.halfedges[f, :3 * T].cpu())
            assert teq(res.normals[j, :T], ref.normals[f, :T].cpu())
        f0 += batch.shape[0]
    assert f0 == 4


SEG_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "segments.npz")


def _seg_golden():
    with np.load(SEG_PATH) as z:
        return {k: z[k] for k in z.files}


@pytest.mark.parametrize("scene", ["room", "frag"])
@pytest.mark.parametrize("ptp", [0.0, 0.01])
@pytest.mark.parametrize("device_mesh", [False, True])
def test_golden_region_growing(fe, scene, ptp, device_mesh):
    """grow_segments (union-find components on the GPU) == the reference's
    region_growing_task membership for every label: same segments, same order, same
    sorted members (tests/golden/make_segments_golden.py), NumPy and device meshes."""
    g = _seg_golden()
    mesh = fe.HalfEdgeMesh(points=g[f"{scene}_points"], triangles=g[f"{scene}_triangles"],
                           halfedges=g[f"{scene}_halfedges"])
    groups = g[f"{scene}_groups"]
    if device_mesh:
        mesh = fe.HalfEdgeMesh(points=torch.from_numpy(mesh.points).cuda(),
                               triangles=torch.from_numpy(mesh.triangles).cuda(),
                               halfedges=torch.from_numpy(mesh.halfedges).cuda())
        groups = torch.from_numpy(groups).cuda()
    params = fe.SegmentationParams(l_max=0.08, ang_min=0.9, ptp_max=ptp,
                                   tri_min=int(g[f"{scene}_tri_min"]))
    for lab in range(len(g["dominant"])):
        got = fe.grow_segments(mesh, groups, lab, g["dominant"][lab], params)
        key = f"{scene}_ptp{ptp:g}_label{lab}"
        exp = np.split(g[key + "_members"], np.cumsum(g[key + "_lengths"])[:-1]) \
            if len(g[key + "_lengths"]) else []
        assert len(got) == len(exp), (lab, len(got), len(exp))
        for a, b in zip(got, exp):
            a = a.cpu().numpy() if isinstance(a, torch.Tensor) else a
            assert np.array_equal(a, b)


def test_grow_segment_kernel_drop_in(fe):
    """_kernels.grow_segment == the oracle's (== _native.pyx:170-222) on single seeds:
    same sorted members, same visited updates, rejected triangles stay seedable."""
    from paper_2007_12065_b200 import _kernels
    g = _seg_golden()
    pts, tris, he, groups = (g["frag_points"], g["frag_triangles"], g["frag_halfedges"],
                             g["frag_groups"])
    rng = np.random.default_rng(3)
    for ptp in (0.0, 0.004, 0.02):
        v_ref = np.zeros(len(tris), np.uint8)
        v_gpu = np.zeros(len(tris), np.uint8)
        cands = np.nonzero(groups != 255)[0]
        for seed in rng.choice(cands, 25, replace=False):
            if v_ref[seed]:
                continue
            lab = int(groups[seed])
            anchor = pts[tris[seed]].mean(axis=0)
            nrm = g["dominant"][lab]
            a = fo.grow_segment(tris, he, pts, groups, v_ref, int(seed), lab, anchor, nrm, ptp)
            b = _kernels.grow_segment(tris, he, pts, groups, v_gpu, int(seed), lab, anchor, nrm,
                                      ptp)
            assert np.array_equal(a, b) and np.array_equal(v_ref, v_gpu)


def test_extract_planar_segment(fe):
    g = _seg_golden()
    mesh = fe.HalfEdgeMesh(points=g["room_points"], triangles=g["room_triangles"],
                           halfedges=g["room_halfedges"])
    groups = g["room_groups"]
    seed = int(np.nonzero(groups == 2)[0][0])
    visited = np.zeros(len(groups), np.uint8)
    m = fe.extract_planar_segment(seed, mesh, groups, g["dominant"][2], 0.01, visited)
    v2 = np.zeros(len(groups), np.uint8)
    exp = fo.grow_segment(mesh.triangles, mesh.halfedges, mesh.points, groups, v2, seed, 2,
                          mesh.points[mesh.triangles[seed]].mean(axis=0), g["dominant"][2], 0.01)
    assert np.array_equal(m, exp) and np.array_equal(visited, v2) and len(m) > 100


@pytest.mark.parametrize("lap_it,src", [(0, torch.float32), (1, torch.float32), (2, torch.float32),
                                        (3, torch.float64), (4, torch.float64)])
def test_profiled_eager_and_graph_agree(fe, lap_it, src):
    """opcfe_front_end_profiled (stage events), opcfe_front_end eagerly and under a CUDA
    graph give identical outputs for odd / even Laplacian pass counts (the ping-pong
    ends in the output buffer), staged f64 input and no Laplacian."""
    frames = fe.synthetic.config_c5_frames(2)[:, :150, :230]
    lap = fe.LaplacianParams(1.0, 3, lap_it) if lap_it else None
    bil = fe.BilateralParams(0.1, 0.15, 3, 3)
    outs = []
    for mode in ("serial", "eager", "graph"):
        eng = fe.FrontEnd(150, 230, 2, laplacian=lap, bilateral=bil, src_dtype=src,
                          graph=mode == "graph")
        eng.src.copy_(torch.from_numpy(frames).to(eng.src.dtype).cuda().reshape(eng.src.shape))
        if mode == "serial":
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
            for e in ev:
                e.record()
            eng.launch_profiled(ev)
        else:
            eng.launch()
            eng.launch()   # graph: capture + replay
        torch.cuda.synchronize()
        r = eng.result()
        outs.append((r.points.clone(), r.triangles.clone(), r.halfedges.clone(),
                     r.normals.clone(), list(r.n_tri)))
    for o in outs[1:]:
        assert o[4] == outs[0][4]
        assert teq(o[0], outs[0][0])
        for f, T in enumerate(o[4]):        # live rows only (capacity rows are scratch)
            assert teq(o[1][f, :T], outs[0][1][f, :T])
            assert teq(o[2][f, :3 * T], outs[0][2][f, :3 * T])
            assert teq(o[3][f, :T], outs[0][3][f, :T])


def test_large_frame_topology_closed_form(fe):
    """A 4000 x 6000 frame (24 M points, 48 M GIDs) through the fused front end, checked on
    the device against the closed forms of SURVEY.md Appendix A (size-independent
    properties of the reference's algorithm, mesh.py:58-135): validity from the smoothed
    grid's NaN mask, trimap = cumsum - 1, triangles (p3,p2,p1) / (p1,p4,p3) in GID
    order, twins 3*trimap[nbr] + k, every twin an involution, unit normals, and the l_max
    flag against fp64 edge lengths."""
    M, N = 4000, 6000
    g = torch.Generator(device="cuda").manual_seed(5)
    u = torch.arange(M, device="cuda", dtype=torch.float32)[:, None].expand(M, N)
    v = torch.arange(N, device="cuda", dtype=torch.float32)[None, :].expand(M, N)
    opc = torch.stack([v * 2e-3, -u * 2e-3, 0.3 * torch.sin(u * 1e-3) * torch.cos(v * 7e-4)], -1)
    opc = opc + 5e-4 * torch.randn((M, N, 3), generator=g, device="cuda")
    opc[torch.rand((M, N), generator=g, device="cuda") < 0.02] = float("nan")
    eng = fe.FrontEnd(M, N, 1, laplacian=fe.LaplacianParams(1.0, 3, 2),
                      bilateral=fe.BilateralParams(0.1, 0.15, 3, 2), l_max=4e-3)
    res = eng.run(opc[None])
    torch.cuda.synchronize()
    pts = res.points[0]
    ok = torch.isfinite(pts).all(-1)
    assert torch.equal(ok, torch.isfinite(opc).all(-1))           # NaN mask invariance
    p1, p2, p3, p4 = ok[:-1, :-1], ok[:-1, 1:], ok[1:, 1:], ok[1:, :-1]
    valid = torch.stack([p1 & p2 & p3, p1 & p3 & p4], -1).reshape(-1)
    T = int(valid.sum())
    assert res.n_tri[0] == T
    trimap = torch.where(valid, torch.cumsum(valid, 0) - 1, torch.full_like(valid, -1, dtype=torch.int64))
    assert torch.equal(res.trimap[0], trimap)
    gid = torch.nonzero(valid).squeeze(1)
    q, k = gid // 2, gid % 2
    qu, qv = q // (N - 1), q % (N - 1)
    i1 = qu * N + qv
    i2, i4 = i1 + 1, i1 + N
    i3 = i4 + 1
    tris = torch.where((k == 0)[:, None], torch.stack([i3, i2, i1], 1), torch.stack([i1, i4, i3], 1))
    assert torch.equal(res.triangles[0, :T], tris)
    # twins: k = 0 -> [(u,v+1,1), (u-1,v,1), (u,v,0+1)]; k = 1 -> [(u,v-1,0), (u+1,v,0), (u,v,0)]
    tm = trimap.view(M - 1, N - 1, 2)
    def nbr(du, dv, kk):
        uu, vv = qu + du, qv + dv
        inside = (uu >= 0) & (uu < M - 1) & (vv >= 0) & (vv < N - 1)
        t = tm[uu.clamp(0, M - 2), vv.clamp(0, N - 2), kk]
        return torch.where(inside & (t >= 0), t, torch.full_like(t, -1))
    first = k == 0
    e0 = torch.where(first, nbr(0, 1, 1), nbr(0, -1, 0))
    e1 = torch.where(first, nbr(-1, 0, 1), nbr(1, 0, 0))
    e2 = torch.where(first, nbr(0, 0, 1), nbr(0, 0, 0))
    he = torch.stack([torch.where(e >= 0, 3 * e + j, e) for j, e in enumerate((e0, e1, e2))], 1)
    got = res.halfedges[0, :3 * T]
    assert torch.equal(got, he.reshape(-1))
    linked = got >= 0
    assert torch.equal(got[got[linked]], torch.nonzero(linked).squeeze(1))
    n = res.normals[0, :T]
    assert torch.isfinite(n).all() and (n.norm(dim=1) - 1).abs().max() < 1e-6
    P = pts.reshape(-1, 3).double()
    a, b, c = P[tris[:, 0]], P[tris[:, 1]], P[tris[:, 2]]
    def norm(d):  # np.linalg.norm's order: sqrt((dx^2 + dy^2) + dz^2)
        return ((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]).sqrt()
    e = torch.maximum(norm(b - a), torch.maximum(norm(c - b), norm(a - c)))
    flag = res.lmax_mask[0, :T].bool()
    assert 0 < int(flag.sum()) < T
    assert torch.equal(flag, e > 4e-3)


@pytest.mark.parametrize("iters", [1, 2, 3, 6])
def test_laplacian_invalid_vertices_bit_identical(fe, iters):
    """Passes 2..L run on a sentinel-encoded grid (laplacian.cu); every non-finite vertex
    must still come back exactly as given (_fallback.py:111-115: a centre with a NaN
    component is copied) -- canonical NaN, partial NaN, other NaN payloads, -NaN -- and
    must not leak into its neighbours."""
    rng = np.random.default_rng(iters)
    M, N = 37, 52
    opc = (grid_opc(M, N) * 0.01 + rng.normal(scale=0.002, size=(M, N, 3))).astype(np.float32)
    bits = opc.view(np.uint32)
    cells = rng.choice(M * N, size=70, replace=False)
    kinds = []
    for i, cell in enumerate(cells):
        u, v = divmod(int(cell), N)
        kind = i % 7
        if kind == 0:
            bits[u, v, :] = 0x7fc00000                      # canonical NaN
        elif kind == 5:
            bits[u, v, :] = 0x7fffffff                      # the GPU's arithmetic NaN
        elif kind == 6:
            bits[u, v, :] = [0x7fc00000, 0x7fc00001, 0x7fc00000]  # mixed payloads
        elif kind == 1:
            bits[u, v, 1] = 0x7fc00000                      # partial NaN
        elif kind == 2:
            bits[u, v, :] = 0x7fc00123                      # NaN payload
        elif kind == 3:
            bits[u, v, :] = 0xffc00000                      # -NaN
        else:
            bits[u, v, 2] = 0x7fa00000                      # partial signalling NaN
        kinds.append((u, v))
    lap = fe.LaplacianParams(1.0, 3, iters)
    _, res = _engine_run(fe, opc, lap, None)
    got = res.points[0].cpu().numpy()
    for u, v in kinds:
        assert np.array_equal(got[u, v].view(np.uint32), opc[u, v].view(np.uint32)), (u, v)
    with np.errstate(invalid="ignore"):                  # signalling NaN -> f64
        ref = c_oracle.laplacian_filter(opc.astype(np.float64), 1.0, 3, iters)
        got64 = got.astype(np.float64)
    assert_vertices_close(got64, ref)


@pytest.mark.parametrize("iters", [2, 5])
def test_laplacian_coincident_neighbours(fe, iters):
    """Duplicated vertices (|d| = 0: the reference skips the pair, _native.pyx:262-266).
    The packed passes see w = inf there and recompute that point by the scalar rule."""
    rng = np.random.default_rng(11 + iters)
    M, N = 40, 70
    opc = (grid_opc(M, N) * 0.01 + rng.normal(scale=0.002, size=(M, N, 3))).astype(np.float32)
    for u, v in rng.integers(1, [M - 2, N - 2], size=(40, 2)):
        opc[u, v + 1] = opc[u, v]                        # right neighbour coincident
        opc[u + 1, v] = opc[u, v]                        # and the one below
    opc[5:9, 10:14] = opc[5, 10]                         # a 4x4 block of one point
    opc[rng.random((M, N)) < 0.03] = np.nan
    _, res = _engine_run(fe, opc, fe.LaplacianParams(1.0, 3, iters), None)
    ref = c_oracle.laplacian_filter(opc.astype(np.float64), 1.0, 3, iters)
    assert_vertices_close(res.points[0].cpu().numpy(), ref)


def _frame_view(res, f):
    from paper_2007_12065_b200.frontend import FrontEndResult
    sl = slice(f, f + 1)
    return FrontEndResult(points=res.points[sl], triangles=res.triangles[sl],
                          trimap=res.trimap[sl],
                          halfedges=None if res.halfedges is None else res.halfedges[sl],
                          normals=None if res.normals is None else res.normals[sl],
                          lmax_mask=None if res.lmax_mask is None else res.lmax_mask[sl],
                          n_tri=[res.n_tri[f]], grid_shape=res.grid_shape)


@pytest.mark.parametrize("seed", range(40))
def test_front_end_randomised(fe, seed):
    """Randomised configurations through the fused front end, per-stage against the oracle,
    every frame of a 1..3-frame batch: odd shapes (tile edges, N % 4 != 0 -> staged
    input), NaN fractions up to 40 %, duplicated vertices, Laplacian 0..6 passes (scalar /
    packed / last-pass restore), kernel sizes 3, 5 and 7, bilateral 0..3 iterations at
    random sigmas, random l_max."""
    rng = np.random.default_rng(1000 + seed)
    M, N = int(rng.integers(3, 170)), int(rng.integers(3, 170))
    F = int(rng.integers(1, 4))
    frames = []
    for f in range(F):
        opc = grid_opc(M, N) * rng.uniform(0.002, 0.05)
        opc[..., 2] = rng.normal(0, 0.01, (M, N)) + 0.2 * np.sin(np.arange(N) / 9.0)[None, :]
        opc += rng.normal(scale=rng.uniform(0, 0.004), size=opc.shape)
        for u, v in rng.integers(0, [max(1, M - 1), max(1, N - 1)],
                                 size=(int(rng.integers(0, 6)), 2)):
            opc[u, min(v + 1, N - 1)] = opc[u, v]
        opc[rng.random((M, N)) < rng.uniform(0, 0.4)] = np.nan
        frames.append(opc.astype(np.float32))
    k_lap = int(rng.choice([3, 3, 3, 5, 7]))
    lap = fe.LaplacianParams(float(rng.uniform(0.3, 1.0)), k_lap, int(rng.integers(1, 7))) \
        if rng.random() < 0.85 and min(M, N) >= k_lap else None
    k_bil = int(rng.choice([3, 3, 3, 5, 7]))
    bil = fe.BilateralParams(float(rng.uniform(0.02, 0.3)), float(rng.uniform(0.08, 0.5)), k_bil,
                             int(rng.integers(1, 4))) if rng.random() < 0.75 else None
    l_max = float(rng.uniform(0.001, 0.05)) if rng.random() < 0.5 else None
    _, res = _engine_run(fe, np.stack(frames), lap, bil, l_max, frames=F)
    for f in range(F):
        _per_stage_check(fe, frames[f], lap, bil, l_max, _frame_view(res, f))


@pytest.mark.parametrize("seed", range(12))
def test_drop_in_api_randomised(fe, seed):
    """The reference-facing functions on random float64 grids (odd shapes, NaN, duplicated
    vertices) against the NumPy restatement of the reference (oracle/flatpoly_oracle.py):
    topology and fp64 normals / FC data bit-exact, Laplacian and bilateral within 1e-5."""
    rng = np.random.default_rng(500 + seed)
    M, N = int(rng.integers(5, 90)), int(rng.integers(5, 90))
    opc = grid_opc(M, N) * rng.uniform(0.003, 0.03)
    opc[..., 2] = rng.normal(0, 0.005, (M, N))
    opc += rng.normal(scale=rng.uniform(0, 0.003), size=opc.shape)
    opc[rng.integers(0, M), :] = opc[rng.integers(0, M), :]       # a duplicated row
    opc[rng.random((M, N)) < rng.uniform(0, 0.3)] = np.nan
    k = int(rng.choice([3, 5]))
    lp = fe.LaplacianParams(float(rng.uniform(0.2, 1.0)), k, int(rng.integers(1, 5)))
    sm = fe.laplacian_filter_opc(opc, lp)
    assert sm.dtype == np.float64 and sm.shape == opc.shape
    assert_vertices_close(sm, fo.laplacian_filter(opc, lp.lam, lp.kernel_size, lp.iterations))
    tris, trimap = fe.extract_triangles_opc(sm)
    rt, rtm = fo.extract_triangles_opc(sm)
    assert np.array_equal(tris, rt) and np.array_equal(trimap, rtm)
    assert np.array_equal(fe.extract_halfedges_opc(trimap, M, N),
                          fo.extract_halfedges_opc(rtm, M, N))
    mesh = fe.mesh_from_opc(sm)
    assert same(mesh.normals, fo.triangle_normals(sm.reshape(-1, 3), rt))
    cen, nrm = fe.compute_fc_triangle_data(sm)
    rc, rn = fo.compute_fc_triangle_data(sm)
    assert same(cen, rc) and same(nrm, rn)
    bp = fe.BilateralParams(float(rng.uniform(0.03, 0.2)), float(rng.uniform(0.1, 0.4)),
                            int(rng.choice([3, 5])), 1)
    got = fe.bilateral_filter_opc(sm, bp, trimap)
    ref = fo.bilateral_filter_opc(sm, bp.sigma_length, bp.sigma_angle, bp.kernel_size,
                                  bp.iterations)
    assert_normals_close(got, ref)


@pytest.mark.parametrize("scale", [1e-4, 1.0, 3e3])
def test_front_end_normals_exact_at_scale(fe, scale):
    """Mesh normals of the fp32 pipeline without bilateral are float32(reference fp64
    normal) exactly (quad_extras_kernel: rsqrt + multiply, exact divide / sqrt only near
    an fp32 rounding midpoint) -- 1.2 M triangles of random shapes per scale."""
    rng = np.random.default_rng(int(scale * 1000) % 997)
    M, N = 700, 900
    opc = grid_opc(M, N) * scale * 0.01
    opc += rng.normal(scale=scale * 0.006, size=opc.shape)
    opc[rng.random((M, N)) < 0.05] = np.nan
    opc = opc.astype(np.float32)
    _, res = _engine_run(fe, opc, None, None, l_max=scale * 0.02)
    T = res.n_tri[0]
    sm = opc.astype(np.float64)
    tris, _, _ = c_oracle.triangulate(sm)
    assert T == len(tris) > 1_000_000
    ref = c_oracle.triangle_normals(sm, tris).astype(np.float32)
    assert same(res.normals[0, :T].cpu().numpy(), ref)
    assert np.array_equal(res.lmax_mask[0, :T].cpu().numpy().astype(bool),
                          c_oracle.max_edge_mask(sm, tris, scale * 0.02))


@pytest.mark.parametrize("cfg", ["lap+bil", "lap+lmax", "f64+bil+lmax", "nolap"])
def test_kernel_launch_count_matches_graph(fe, cfg):
    """bench.py's gpu_launches = FrontEnd.kernel_launches x steps: the count equals the
    kernel nodes of the captured front-end graph, and every node is a libopcfe kernel."""
    from cuda.bindings import driver as drv
    M, N = 70, 96
    opc = grid_opc(M, N) * 0.01
    opc[5, 7] = np.nan
    kw = dict(laplacian=fe.LaplacianParams(1.0, 3, 3), bilateral=fe.BilateralParams())
    dtype = torch.float32
    if cfg == "lap+lmax":
        kw.update(bilateral=None, l_max=0.02)
    elif cfg == "f64+bil+lmax":
        kw.update(l_max=0.02)
        dtype = torch.float64
    elif cfg == "nolap":
        kw.update(laplacian=None)
    eng = fe.FrontEnd(M, N, 2, src_dtype=dtype, graph=False, **kw)
    eng.src.copy_(torch.from_numpy(opc).to("cuda", dtype).expand(2, M, N, 3))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        eng._launch(s)                                   # warm-up outside the capture
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph(keep_graph=True)
    with torch.cuda.graph(g, stream=s):
        eng._launch(s)
    graph = drv.CUgraph(g.raw_cuda_graph())
    err, _, n = drv.cuGraphGetNodes(graph, 0)
    assert err == drv.CUresult.CUDA_SUCCESS
    err, nodes, n = drv.cuGraphGetNodes(graph, n)
    names = []
    for node in nodes[:n]:
        err, kind = drv.cuGraphNodeGetType(node)
        if kind == drv.CUgraphNodeType.CU_GRAPH_NODE_TYPE_KERNEL:
            err, params = drv.cuGraphKernelNodeGetParams(node)
            err, name = drv.cuFuncGetName(params.func)
            names.append(name.decode() if isinstance(name, bytes) else str(name))
    assert len(names) == eng.kernel_launches, names
    assert all("opcfe" in nm for nm in names), names


@pytest.mark.parametrize("offset", [0.0, 50.0, 400.0])
def test_bilateral_far_from_origin(fe, offset):
    """A scene far from the coordinate origin with a small sigma_length: fp32 centroids
    carry an absolute rounding ~|c| 2^-24, which tile-relative centroids keep out of the
    weights (without them, 50 m at 13 mm spacing and sl = 2 cm broke 1e-5)."""
    opc = fe.synthetic.room_scene(n=300, noise=0.002, seed=3)
    opc = opc + np.array([offset, -0.5 * offset, 0.1 * offset])
    lap = fe.LaplacianParams(1.0, 3, 2)
    bil = fe.BilateralParams(0.02, 0.15, 3, 3)
    _, res = _engine_run(fe, opc, lap, bil)
    _per_stage_check(fe, opc, lap, bil, None, res)


@pytest.mark.parametrize("offset", [0.0, 300.0])
def test_drop_in_bilateral_far_from_origin(fe, offset):
    """The float64 drop-in (_kernels.bilateral_iterate / bilateral_filter_opc) takes its
    centroids in float64 and subtracts the tile origin in fp64, so a scene hundreds of
    metres out keeps the 1e-5 contract at a small sigma_length."""
    opc = fe.synthetic.room_scene(n=160, noise=0.002, seed=8) + np.array([offset, 0.3 * offset, 0.0])
    bp = fe.BilateralParams(0.03, 0.2, 3, 2)
    got = fe.bilateral_filter_opc(opc, bp)
    ref = fo.bilateral_filter_opc(opc, bp.sigma_length, bp.sigma_angle, bp.kernel_size,
                                  bp.iterations)
    assert_normals_close(got, ref)
    cen, nrm = fo.compute_fc_triangle_data(opc)
    g1 = fe._kernels.bilateral_iterate(cen, nrm, 0.03, 0.2, 3, 1)
    assert_normals_close(g1, fo.bilateral_iterate(cen, nrm, 0.03, 0.2, 3, 1))


@pytest.mark.parametrize("shape", [(6, 9001), (4100, 5)])
def test_front_end_wide_and_tall(fe, shape):
    """The fused front end on rows wider than one triangulation scan segment (4096 quads)
    and on a tall 4-quad-wide grid (partial TMA boxes on every row), 2-frame batch,
    per-stage against the oracle."""
    M, N = shape
    rng = np.random.default_rng(M + N)
    frames = []
    for _ in range(2):
        opc = grid_opc(M, N) * 0.01
        opc[..., 2] = rng.normal(0, 0.01, (M, N))
        opc[rng.random((M, N)) < 0.1] = np.nan
        frames.append(opc.astype(np.float32))
    lap = fe.LaplacianParams(1.0, 3, 3)
    bil = fe.BilateralParams(0.1, 0.15, 3, 2)
    _, res = _engine_run(fe, np.stack(frames), lap, bil, 0.02, frames=2)
    for f in range(2):
        _per_stage_check(fe, frames[f], lap, bil, 0.02, _frame_view(res, f))


def test_front_end_many_frames(fe):
    """A 300-frame batch of small distinct frames (C1-style batching): frame strides of
    every stage, per-stage against the oracle on the first, last and 8 random frames."""
    M, N, F = 20, 27, 300
    rng = np.random.default_rng(300)
    frames = []
    for _ in range(F):
        opc = grid_opc(M, N) * rng.uniform(0.005, 0.03)
        opc[..., 2] = rng.normal(0, 0.01, (M, N))
        opc[rng.random((M, N)) < rng.uniform(0, 0.3)] = np.nan
        frames.append(opc.astype(np.float32))
    lap = fe.LaplacianParams(0.8, 3, 2)
    bil = fe.BilateralParams(0.05, 0.2, 3, 2)
    _, res = _engine_run(fe, np.stack(frames), lap, bil, 0.03, frames=F)
    for f in [0, F - 1] + [int(x) for x in rng.choice(np.arange(1, F - 1), 8, replace=False)]:
        _per_stage_check(fe, frames[f], lap, bil, 0.03, _frame_view(res, f))


@pytest.mark.parametrize("level", [2, 4])
def test_fastga_on_own_accumulator(fe, level):
    """build_accumulator (host gauss_sphere, bit-identical structure) + the GPU search:
    the same cells and votes as the reference-built structure, and the reference's own
    accumulator tests (test_accumulator.py:92-172) on it."""
    g = FASTGA[f"level{level}"]
    ga = fe.build_accumulator(level)
    slope, icpt, wlo, whi = g["model"]
    ref = fe._kernels.find_cells(g["queries"], g["ids"], g["cell_normals"], g["neighbors"],
                                 slope, icpt, int(wlo), int(whi))
    assert np.array_equal(fe.find_cell_indices(ga, g["queries"]), ref)
    counts = fe.integrate_normals(ga, g["mesh_normals"], sample_pct=0.12)
    assert counts is ga.counts and counts.sum() == g["counts"].sum()
    for idx in (0, 17, ga.num_cells // 2, ga.num_cells - 1):
        assert fe.find_cell_index(ga, ga.normals[idx]) == idx
        assert fe.find_cell_index(ga, 3.0 * ga.normals[idx]) == idx
    with pytest.raises(ValueError):
        fe.find_cell_index(ga, np.zeros(3))
    rng = np.random.default_rng(level)
    q = rng.normal(size=(5000, 3))
    q /= np.linalg.norm(q, axis=1)[:, None]
    got = fe.find_cell_indices(ga, q)
    true = np.argmax(q @ ga.normals.T, axis=1)
    agree = got == true
    assert agree.mean() >= 0.999
    for i in np.nonzero(~agree)[0]:
        assert got[i] in ga.neighbors[true[i]]
    ga2 = fe.build_accumulator(level)                 # fresh zero counts, shared structure
    assert fe.integrate_normals(ga2, np.empty((0, 3))).sum() == 0
    assert fe.find_cell_indices(ga2, np.empty((0, 3))).shape == (0,)
    fe.integrate_normals(ga2, np.tile(ga2.normals[42], (9, 1)))
    assert ga2.counts[42] == 9 and ga2.counts.sum() == 9
    ga3 = fe.build_accumulator(level)
    fe.integrate_normals(ga3, np.tile(ga3.normals[7], (10, 1)), sample_pct=0.25)
    assert ga3.counts.sum() == 3                      # rows 0, 4, 8
    ga4 = fe.build_accumulator(level)
    n = np.tile(ga4.normals[3], (5, 1))
    n[1] = np.nan
    n[3, 2] = np.inf
    fe.integrate_normals(ga4, n)
    assert ga4.counts.sum() == 3


@pytest.mark.parametrize("n,offset", [(0, 0), (1, 0), (7, 1), (4_141_202, 0), (4_141_203, 1),
                                      (1000, 0)])
def test_trimap_stats(n, offset):
    """opcfe_trimap_stats (count of entries >= 0, max(-1, largest)) against NumPy: odd
    lengths, a 8-B (not 16-B) aligned start, all-invalid maps."""
    from paper_2007_12065_b200 import _ops
    rng = np.random.default_rng(n)
    tm = np.where(rng.random(n + offset) < 0.7, rng.integers(0, 1 << 40, n + offset), -1)
    if n == 1000:
        tm[:] = -1
    d = torch.from_numpy(tm).cuda()[offset:]
    assert _ops.trimap_stats(d) == (int((tm[offset:] >= 0).sum()),
                                    int(max(-1, tm[offset:].max())) if n else -1)
