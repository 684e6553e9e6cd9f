"""Single-process multi-device driver (distributed.MultiDevicePipeline) on the GPU box.

The box has one GPU, so the driver runs two independent pipelines on device 0 from two
host threads (its own streams, pinned buffers and graphs each): the per-device shards
must cover the batch exactly once and every frame's outputs must equal a single
pipeline's.  (On an 8-GPU node `devices=None` takes every visible device.)
"""

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


def teq(a, b):
    a, b = a.contiguous(), b.contiguous()
    if a.is_floating_point():
        return torch.equal(torch.isnan(a), torch.isnan(b)) and \
            torch.equal(torch.nan_to_num(a), torch.nan_to_num(b))
    return torch.equal(a, b)


@pytest.mark.parametrize("F,devs", [(5, [0, 0]), (7, [0, 0, 0]), (1, [0, 0])])
def test_multi_device_pipeline_matches_single(F, devs):
    import paper_2007_12065_b200 as fe
    from paper_2007_12065_b200.distributed import MultiDevicePipeline
    frames = fe.synthetic.config_c5_frames(F)[:, :72, :100]
    M, N = frames.shape[1:3]
    lap, bil = fe.LaplacianParams(1.0, 3, 2), fe.BilateralParams(0.1, 0.15, 3, 2)
    host = torch.from_numpy(frames).pin_memory()
    multi = MultiDevicePipeline(M, N, devices=devs, laplacian=lap, bilateral=bil,
                                frames_per_slot=2)
    parts = multi.run(host)
    single = fe.HostPipeline(M, N, laplacian=lap, bilateral=bil, frames_per_slot=2)
    ref = single.run(host)
    covered = []
    for (a, b), res in zip(multi.shards, parts):
        covered += list(range(a, b))
        for j in range(b - a):
            f = a + j
            T = ref.n_tri[f]
            assert res.n_tri[j] == T
            assert teq(res.points[j], ref.points[f])
            assert teq(res.triangles[j, :T], ref.triangles[f, :T])
            assert teq(res.halfedges[j, :3 * T], ref.halfedges[f, :3 * T])
            assert teq(res.normals[j, :T], ref.normals[f, :T])
            assert teq(res.trimap[j], ref.trimap[f])
    assert covered == list(range(F))
    assert multi.h2d_bytes == host.numel() * 8
