"""Pin the CPU oracle (NumPy and C restatements) to the reference's golden vectors.

The golden files were produced by the real reference (tests/golden/make_golden.py).
These tests run without a GPU.
"""

import os

import numpy as np
import pytest

from conftest import load_golden
from oracle import c_oracle
from oracle import flatpoly_oracle as fo

TOPO = load_golden("topology")
LAP = load_golden("laplacian")
BIL = load_golden("bilateral")
FE = load_golden("frontend")


def same_f64(a, b):
    """bit-identical including NaN positions"""
    a = np.asarray(a)
    b = np.asarray(b)
    return a.shape == b.shape and np.array_equal(np.isnan(a), np.isnan(b)) and \
        np.array_equal(np.nan_to_num(a), np.nan_to_num(b))


@pytest.mark.parametrize("case", sorted(TOPO))
def test_topology_numpy_oracle(case):
    g = TOPO[case]
    tris, trimap = fo.extract_triangles_opc(g["opc"])
    assert np.array_equal(tris, g["triangles"])
    assert np.array_equal(trimap, g["trimap"])
    M, N = g["opc"].shape[:2]
    assert np.array_equal(fo.extract_halfedges_opc(trimap, M, N), g["halfedges"])
    assert same_f64(fo.triangle_normals(g["opc"].reshape(-1, 3), tris), g["normals"])
    cen, nrm = fo.compute_fc_triangle_data(g["opc"])
    assert same_f64(cen, g["fc_centroids"]) and same_f64(nrm, g["fc_normals"])


@pytest.mark.parametrize("case", sorted(TOPO))
def test_topology_c_oracle(case):
    g = TOPO[case]
    tris, trimap, he = c_oracle.triangulate(g["opc"])
    assert np.array_equal(tris, g["triangles"])
    assert np.array_equal(trimap, g["trimap"])
    assert np.array_equal(he, g["halfedges"])
    assert same_f64(c_oracle.triangle_normals(g["opc"], tris), g["normals"])
    cen, nrm = c_oracle.compute_fc_triangle_data(g["opc"])
    assert same_f64(cen, g["fc_centroids"]) and same_f64(nrm, g["fc_normals"])


@pytest.mark.parametrize("case", sorted(LAP))
def test_laplacian_oracles_bit_exact(case):
    g = LAP[case]
    lam, k, it = g["params"]
    a = fo.laplacian_filter(g["opc"], lam, int(k), int(it))
    b = c_oracle.laplacian_filter(g["opc"], lam, int(k), int(it))
    assert same_f64(a, g["out"])
    assert same_f64(b, g["out"])
    if "out_native" in g:
        assert same_f64(b, g["out_native"])


@pytest.mark.parametrize("case", sorted(c for c in BIL if c.startswith("iter")))
def test_bilateral_iterate_oracles(case):
    g = BIL[case]
    sl, sa, k, it = g["params"]
    a = fo.bilateral_iterate(g["centroids"], g["normals"], sl, sa, int(k), int(it))
    b = c_oracle.bilateral_iterate(g["centroids"], g["normals"], sl, sa, int(k), int(it))
    for ref in (g["out"], g["out_native"]):
        assert np.array_equal(np.isnan(a), np.isnan(ref))
        assert np.nanmax(np.abs(a - ref)) < 1e-14      # exp: 1-ulp libm vs SIMD
        assert np.nanmax(np.abs(b - ref)) < 1e-14


@pytest.mark.parametrize("case", sorted(c for c in BIL if not c.startswith("iter")))
def test_bilateral_filter_opc_oracle(case):
    g = BIL[case]
    sl, sa, k, it = g["params"]
    out = fo.bilateral_filter_opc(g["opc"], sl, sa, int(k), int(it))
    assert out.shape == g["out"].shape
    assert np.nanmax(np.abs(out - g["out"])) < 1e-14


@pytest.mark.parametrize("impl", [fo, c_oracle], ids=["numpy", "c"])
def test_front_end_room(impl):
    g = FE["room"]
    lam, k, it = g["lap"]
    sl, sa, kb, itb = g["bil"]
    r = impl.front_end(g["opc"], (lam, int(k), int(it)), (sl, sa, int(kb), int(itb)))
    assert same_f64(r["smoothed"], g["smoothed"])
    assert np.array_equal(r["triangles"], g["triangles"])
    assert np.array_equal(r["trimap"], g["trimap"])
    assert np.array_equal(r["halfedges"], g["halfedges"])
    assert np.max(np.abs(r["normals"] - g["normals"])) < 1e-14
    plain = impl.triangle_normals(r["smoothed"].reshape(-1, 3), r["triangles"])
    assert same_f64(plain, g["mesh_normals"])


@pytest.mark.parametrize("impl", [fo, c_oracle], ids=["numpy", "c"])
def test_lmax_mask_matches_group_assignment(impl):
    for case, lmaxes in (("room", (0.05, 0.5)), ("lidar", (0.5,))):
        g = FE[case]
        src = g["smoothed"].reshape(-1, 3)
        keep = g["labels_lmaxinf"] != 255          # triangles the angle filter keeps
        for l_max in lmaxes:
            mask = impl.max_edge_mask(src, g["triangles"], l_max)
            lab = g[f"labels_lmax{l_max}"]
            assert np.array_equal(mask[keep], lab[keep] == 255)
    g = FE["grid3"]
    tris, _ = fo.extract_triangles_opc(g["opc"])
    assert np.all(impl.max_edge_mask(g["opc"].reshape(-1, 3), tris, 0.5)) 
    assert not np.any(impl.max_edge_mask(g["opc"].reshape(-1, 3), tris, 2.0))
    assert np.all(g["labels_lmax0.5"] == 255) and np.all(g["labels_lmax2.0"] == 0)


GROUPS = load_golden("groups")


@pytest.mark.parametrize("impl", [fo, c_oracle], ids=["numpy", "c"])
@pytest.mark.parametrize("case", sorted(GROUPS))
def test_group_assignment_oracles(impl, case):
    g = GROUPS[case]
    l_max, ang = g["params"]
    lab = impl.group_assignment(g["points"], g["triangles"], g["normals"], g["dominant"],
                                l_max, ang)
    assert lab.dtype == np.uint8 and np.array_equal(lab, g["labels"])
    with pytest.raises(ValueError):
        impl.group_assignment(g["points"], g["triangles"], g["normals"], np.zeros((0, 3)),
                              l_max, ang)


FASTGA = load_golden("fastga")


@pytest.mark.parametrize("case", sorted(FASTGA))
def test_fastga_c_oracle(case):
    """C restatement of sfc.s2_id + find_cells + integrate_normals == the reference."""
    g = FASTGA[case]
    slope, icpt, wlo, whi = g["model"]
    assert np.array_equal(c_oracle.s2_id(g["queries"][:2000]), g["s2id"][:2000])
    cells = c_oracle.find_cells(g["queries"], g["ids"], g["cell_normals"], g["neighbors"],
                                slope, icpt, int(wlo), int(whi))
    assert np.array_equal(cells, g["cells"]) and np.array_equal(cells, g["cells_native"])
    counts = c_oracle.integrate_normals(np.zeros(len(g["ids"]), dtype=np.int64),
                                        g["mesh_normals"], g["ids"], g["cell_normals"],
                                        g["neighbors"], slope, icpt, int(wlo), int(whi), 0.12)
    assert np.array_equal(counts, g["counts"])


def test_lidar_front_end():
    g = FE["lidar"]
    lam, k, it = g["lap"]
    r = c_oracle.front_end(g["opc"], (lam, int(k), int(it)), None)
    assert same_f64(r["smoothed"], g["smoothed"])
    assert np.array_equal(r["triangles"], g["triangles"])
    assert np.array_equal(r["halfedges"], g["halfedges"])
    assert same_f64(r["normals"], g["mesh_normals"])


SEG_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "segments.npz")


def seg_golden():
    with np.load(SEG_PATH) as z:
        return {k: z[k] for k in z.files}


def seg_expected(g, scene, ptp, lab):
    key = f"{scene}_ptp{ptp:g}_label{lab}"
    return np.split(g[key + "_members"], np.cumsum(g[key + "_lengths"])[:-1]) \
        if len(g[key + "_lengths"]) else []


@pytest.mark.parametrize("scene", ["room", "frag"])
@pytest.mark.parametrize("ptp", [0.0, 0.01])
def test_region_growing_oracle(scene, ptp):
    """oracle.grow_segments == the reference's region_growing_task membership
    (tests/golden/make_segments_golden.py), every label, planarity check off and on."""
    g = seg_golden()
    for lab in range(len(g["dominant"])):
        got = fo.grow_segments(g[f"{scene}_points"], g[f"{scene}_triangles"],
                               g[f"{scene}_halfedges"], g[f"{scene}_groups"], lab,
                               g["dominant"][lab], ptp, int(g[f"{scene}_tri_min"]))
        exp = seg_expected(g, scene, ptp, lab)
        assert len(got) == len(exp)
        for a, b in zip(got, exp):
            assert np.array_equal(a, b)


# ---------------------------------------------- chains (tests/golden/make_chain_golden.py)
CHAIN = load_golden("chain")


@pytest.mark.parametrize("case", sorted(CHAIN))
def test_c_oracle_chain_pinned(case):
    """The C oracle's fp64 chain (laplacian -> mesh -> bilateral, pipeline.py:125-134)
    equals the reference's own chain: smoothed grid and topology bit-exact, normals to
    exp()'s last ulp (the GPU strict chain is checked against both)."""
    g = CHAIN[case]
    lap = tuple(g["lap"][:1]) + tuple(int(x) for x in g["lap"][1:])
    bil = None
    if g["bil"].size:
        b = g["bil"]
        bil = (float(b[0]), float(b[1]), int(b[2]), int(b[3]))
    r = c_oracle.front_end(g["opc"], lap, bil)
    sm = r["smoothed"]
    assert np.array_equal(np.isnan(sm), np.isnan(g["smoothed"]))
    assert np.array_equal(np.nan_to_num(sm), np.nan_to_num(g["smoothed"]))
    assert np.array_equal(r["trimap"], g["trimap"].astype(np.int64))
    assert int((r["halfedges"] >= 0).sum()) == int(g["n_halfedges_linked"][0])
    n, ref = r["normals"], g["normals"]
    assert np.array_equal(np.isnan(n), np.isnan(ref))
    ok = ~np.isnan(ref).any(1)
    assert np.max(np.linalg.norm(n[ok] - ref[ok], axis=1)) <= 1e-13
    l_max, ang = (float(x) for x in g["seg"])
    lab = c_oracle.group_assignment(r["points"], r["triangles"], n, g["dominant"], l_max, ang)
    assert np.array_equal(lab, g["labels"])
