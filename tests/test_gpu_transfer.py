"""Host <-> device transfers of the NumPy drop-in API (_device.HostTransfer).

Large results come back as NumPy views of pinned host blocks (one DMA into the caller's
array); past the pinned budget they take the staged path into a fresh pageable array.
Both must hand back the same bytes, writeable, independent of later calls; pinned inputs
(a previous call's result) are DMA'd straight to the device.
"""

import gc

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


@pytest.fixture()
def xfer():
    from paper_2007_12065_b200._device import HostTransfer
    return HostTransfer.get(torch.cuda.current_device())


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.int64])
def test_large_result_paths_agree(xfer, dtype):
    g = torch.Generator(device="cuda").manual_seed(7)
    t = (torch.rand((1_500_001, 3), generator=g, device="cuda", dtype=torch.float64) * 1e6).to(dtype)
    ref = t.cpu().numpy()
    a = xfer.to_numpy(t)
    assert a.flags.writeable and a.flags.c_contiguous and a.dtype == ref.dtype
    assert torch.from_numpy(a).is_pinned()
    old = xfer.PINNED_OUT_MB
    try:
        xfer.PINNED_OUT_MB = 0                     # budget exhausted -> staged path
        b = xfer.to_numpy(t)
    finally:
        xfer.PINNED_OUT_MB = old
    assert not torch.from_numpy(b).is_pinned()
    np.testing.assert_array_equal(a, ref)
    np.testing.assert_array_equal(b, ref)
    a[0, 0] = -1                                    # results are the caller's own memory
    c = xfer.to_numpy(t)
    assert c[0, 0] == ref[0, 0] and a[0, 0] == -1


def test_pinned_blocks_are_reused(xfer):
    t = torch.ones((4 << 20,), dtype=torch.float64, device="cuda")
    for _ in range(3):
        xfer.to_numpy(t)
    gc.collect()
    before = torch.cuda.host_memory_stats().get("allocated_bytes.current", 0)
    for _ in range(20):
        a = xfer.to_numpy(t)
        assert a[-1] == 1.0
        del a
    after = torch.cuda.host_memory_stats().get("allocated_bytes.current", 0)
    assert after == before                          # no new pinned blocks per call
    held = xfer.out_bytes
    keep = [xfer.to_numpy(t) for _ in range(3)]     # results alive count against the budget
    assert xfer.out_bytes == held + 3 * (4 << 23)
    view = keep[0][5:]
    del keep
    gc.collect()
    assert xfer.out_bytes == held + (4 << 23)       # a view keeps its block
    del view
    gc.collect()
    assert xfer.out_bytes == held


def test_pinned_input_round_trip(xfer):
    t = torch.arange(3 * 1_000_003, dtype=torch.float64, device="cuda").reshape(-1, 3)
    a = xfer.to_numpy(t)                            # pinned-backed
    assert torch.from_numpy(a).is_pinned()
    d = xfer.to_device(a)
    assert torch.equal(d, t)
    p = np.asarray(a[10:])                          # a view into the pinned block
    assert torch.equal(xfer.to_device(p), t[10:])
    q = np.array(a)                                 # pageable copy: staged path
    assert torch.equal(xfer.to_device(q), t)


def test_dropin_chain_same_with_and_without_pinned_outputs(xfer):
    import paper_2007_12065_b200 as fe
    frame = fe.synthetic.config_c2()
    lp, bp = fe.LaplacianParams(1.0, 3, 3), fe.BilateralParams(0.1, 0.15, 3, 2)

    def chain():
        sm = fe.laplacian_filter_opc(frame, lp)
        mesh = fe.mesh_from_opc(sm)
        n = fe.bilateral_filter_opc(sm, bp, mesh.trimap)
        return sm, mesh.triangles, mesh.halfedges, mesh.trimap, mesh.normals, n

    r1 = chain()
    old, old_min = xfer.PINNED_OUT_MB, xfer.MIN_BYTES
    try:
        xfer.PINNED_OUT_MB = 0
        xfer.MIN_BYTES = 1 << 16                    # force the staged paths at C2 size
        r2 = chain()
    finally:
        xfer.PINNED_OUT_MB, xfer.MIN_BYTES = old, old_min
    for x, y in zip(r1, r2):
        np.testing.assert_array_equal(x, y)
