"""Multi-process (world_size 2, gloo, CPU) tests of the frame-batch sharding plumbing.

The device kernels cannot run here; the data path has no collective anyway, so what
is tested is the host logic every rank runs: contiguous shards that cover the batch
exactly once, max-over-ranks timing and sum-over-ranks bookkeeping.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2007_12065_b200.distributed import shard_range


@pytest.mark.parametrize("n,world", [(512, 1), (512, 2), (512, 8), (7, 3), (2, 4), (0, 2)])
def test_shards_cover_exactly_once(n, world):
    seen = []
    sizes = []
    for r in range(world):
        a, b = shard_range(n, world, r)
        seen.extend(range(a, b))
        sizes.append(b - a)
    assert seen == list(range(n))
    assert max(sizes) - min(sizes) <= 1


def test_bad_rank():
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2007_12065_b200 import distributed as D
        info = D.rank_info()
        frames = np.arange(10 * 4 * 5 * 3, dtype=np.float64).reshape(10, 4, 5, 3)

        def process(chunk):  # stand-in for FrontEnd.run: per-frame "triangle counts"
            return [int(f[0, 0, 0]) for f in chunk]

        start, stop, counts = D.run_sharded(frames, process, batch=3, info=info)
        t = D.max_over_ranks(1.0 + rank)
        total = D.sum_over_ranks(len(counts))
        # real per-frame outputs: every rank meshes its shard of 7 small NaN-holed frames
        # (the front end's CPU restatement stands in for the GPU, which is absent here),
        # results gathered at their global frame offsets
        from oracle import c_oracle
        rng = np.random.default_rng(3)
        opcs = rng.normal(size=(7, 9, 11, 3))
        opcs[rng.random((7, 9, 11)) < 0.2] = np.nan

        def mesh(chunk):
            out = []
            for o in chunk:
                r = c_oracle.front_end(o, (1.0, 3, 2), (0.1, 0.15, 3, 1))
                out.append((r["triangles"], r["halfedges"], r["normals"]))
            return out

        s2, e2, meshes = D.run_sharded(opcs, mesh, batch=2, info=info)
        allm = D.gather_shards(s2, meshes)
        q.put((rank, start, stop, counts, t, total, (s2, e2), allm))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding_and_timing():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=180) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, a0, b0, c0, t0, n0, sh0, m0), (r1, a1, b1, c1, t1, n1, sh1, m1) = out
    assert (a0, b0, a1, b1) == (0, 5, 5, 10)
    assert c0 + c1 == [i * 60 for i in range(10)]      # every frame processed once, in order
    assert t0 == t1 == 2.0                               # max over ranks
    assert n0 == n1 == 10
    assert (sh0, sh1) == ((0, 4), (4, 7))
    # both ranks hold all 7 meshes at their global offsets, equal to one process's
    from oracle import c_oracle
    rng = np.random.default_rng(3)
    opcs = rng.normal(size=(7, 9, 11, 3))
    opcs[rng.random((7, 9, 11)) < 0.2] = np.nan
    for f in range(7):
        r = c_oracle.front_end(opcs[f], (1.0, 3, 2), (0.1, 0.15, 3, 1))
        for m in (m0, m1):
            tri, he, nrm = m[f]
            assert np.array_equal(tri, r["triangles"]) and np.array_equal(he, r["halfedges"])
            assert np.array_equal(np.isnan(nrm), np.isnan(r["normals"]))
            assert np.array_equal(np.nan_to_num(nrm), np.nan_to_num(r["normals"]))
