"""FastGA accumulator structure built by paper_2007_12065_b200.gauss_sphere (host, NumPy)
against the reference's own build (tests/golden/make_accumulator_golden.py): bit-identical
arrays and model scalars at every level 0..7, plus the reference's structural tests
(test_accumulator.py:20-90).  CPU only; the GPU search over these structures is in
tests/test_gpu_parity.py / test_gpu_reference_cases.py."""

import hashlib
import json
import os

import numpy as np
import pytest

from paper_2007_12065_b200 import build_accumulator, gauss_sphere

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLDEN, "accumulator.json")) as f:
        return json.load(f)["levels"]


@pytest.mark.parametrize("level", range(8))
def test_structure_bit_identical_to_reference(golden, level):
    g = golden[str(level)]
    ga = build_accumulator(level)
    assert ga.num_cells == g["cells"] == 20 * 4 ** level
    assert digest(ga.normals.astype(np.float64)) == g["normals_f64"]
    assert digest(ga.s2ids.astype(np.uint64)) == g["s2ids_u64"]
    assert digest(ga.neighbors.astype(np.int64)) == g["neighbors_i64"]
    assert float(ga.model_slope).hex() == g["slope"]
    assert float(ga.model_intercept).hex() == g["intercept"]
    assert [ga.window_lo, ga.window_hi] == g["window"]
    assert ga.counts.dtype == np.int64 and not ga.counts.any()


def test_s2_ids_and_hilbert_match_reference():
    z = np.load(os.path.join(GOLDEN, "s2ids.npz"))
    np.testing.assert_array_equal(gauss_sphere.s2_ids(z["normals"]), z["ids"])
    np.testing.assert_array_equal(gauss_sphere.hilbert_index(z["hx"], z["hy"]), z["hd"])
    with pytest.raises(ValueError):
        gauss_sphere.s2_ids(np.zeros((1, 3)))
    with pytest.raises(ValueError):
        gauss_sphere.s2_ids(np.array([[np.nan, 0, 1.0]]))


def test_hilbert_small_grid_is_a_curve():
    # every cell visited once, consecutive positions are grid neighbours
    n = 16
    x, y = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    d = gauss_sphere.hilbert_index(x.ravel(), y.ravel(), bits=4)
    assert sorted(d.tolist()) == list(range(n * n))
    order = np.argsort(d)
    step = np.abs(np.diff(x.ravel()[order])) + np.abs(np.diff(y.ravel()[order]))
    assert (step == 1).all()


@pytest.mark.parametrize("level,nv,nt", [(0, 12, 20), (1, 42, 80), (2, 162, 320),
                                         (3, 642, 1280), (4, 2562, 5120)])
def test_refinement_counts(level, nv, nt):
    V, F = gauss_sphere.refined_icosahedron(level)
    assert V.shape == (nv, 3) and F.shape == (nt, 3)
    np.testing.assert_allclose(np.linalg.norm(V, axis=1), 1.0, atol=1e-12)


@pytest.mark.parametrize("level", [1, 2, 3])
def test_sixty_cells_with_eleven_neighbors(level):
    nbrs = build_accumulator(level).neighbors
    missing = (nbrs == -1).sum(axis=1)
    assert (missing == 1).sum() == 60 and (missing == 0).sum() == len(nbrs) - 60


def test_neighbors_share_a_vertex_and_are_symmetric():
    V, F = gauss_sphere.refined_icosahedron(2)
    ring = gauss_sphere.one_ring(F, len(V))
    for t in range(len(F)):
        row = ring[t][ring[t] >= 0]
        assert np.all(np.diff(row) > 0) and t not in row
        for nb in row:
            assert set(F[t]) & set(F[nb]) and t in ring[nb]


def test_sorted_window_and_levels():
    ga = build_accumulator(4)
    assert np.all(np.diff(ga.s2ids.astype(np.int64)) > 0)
    idx = np.arange(ga.num_cells, dtype=np.float64)
    err = idx - (ga.model_slope * ga.s2ids.astype(np.float64) + ga.model_intercept)
    assert ga.window_lo <= np.floor(err.min()) and ga.window_hi >= np.ceil(err.max())
    with pytest.raises(ValueError):
        build_accumulator(-1)
    with pytest.raises(ValueError):
        build_accumulator(8)
    a, b = build_accumulator(3), build_accumulator(3)
    assert a.s2ids is b.s2ids and a.counts is not b.counts    # shared structure, own counts
    assert not a.s2ids.flags.writeable


@pytest.mark.parametrize("level", [2, 4])
def test_structure_equals_fastga_golden_arrays(level):
    z = np.load(os.path.join(GOLDEN, "fastga.npz"))
    ga = build_accumulator(level)
    np.testing.assert_array_equal(ga.s2ids, z[f"level{level}/ids"])
    np.testing.assert_array_equal(ga.normals, z[f"level{level}/cell_normals"])
    np.testing.assert_array_equal(ga.neighbors, z[f"level{level}/neighbors"])
    slope, icpt, wlo, whi = z[f"level{level}/model"]
    assert (ga.model_slope, ga.model_intercept, ga.window_lo, ga.window_hi) == \
        (slope, icpt, int(wlo), int(whi))
