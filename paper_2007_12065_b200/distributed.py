"""Frame-batch data parallelism across the GPUs of one node.

Frames are independent units: a batch of frames is split into contiguous chunks, one
per rank (one process per GPU, torch.distributed for the plumbing).  There is NO
collective on the data path -- every rank runs its own FrontEnd on its own frames and
keeps its results; the only collectives are for timing (max over ranks) and
bookkeeping (frame / triangle counts), which work on NCCL or gloo alike.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import torch


@dataclass
class RankInfo:
    rank: int = 0
    world: int = 1
    local_rank: int = 0


def rank_info() -> RankInfo:
    """RANK / WORLD_SIZE / LOCAL_RANK from the torchrun environment (defaults: 1 process)."""
    return RankInfo(int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
                    int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(n_frames: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, stop) of `n_frames` for `rank`; shard sizes differ by at most 1."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(n_frames, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def _reduce(value: float, op, device=None) -> float:
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    dev = device
    if dist.get_backend() != "nccl":
        dev = torch.device("cpu")              # gloo: host tensors
    elif dev is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op)
    return float(t.item())


def max_over_ranks(value: float, device=None) -> float:
    """Job time = the slowest rank's device time (timing rule: max over ranks)."""
    import torch.distributed as dist
    return _reduce(value, dist.ReduceOp.MAX, device)


def sum_over_ranks(value: float, device=None) -> float:
    import torch.distributed as dist
    return _reduce(value, dist.ReduceOp.SUM, device)


def run_sharded(frames, process_batch, batch: int, info: RankInfo | None = None):
    """Run this rank's contiguous shard of `frames` through `process_batch` in batches.

    `frames` is an indexable of F frames (host or device); `process_batch(chunk)` runs the
    front end on a (<= batch, M, N, 3) slice and returns one result per frame (triangle
    counts, meshes, ...).  Returns (start, stop, per-frame results) for this rank: result
    j belongs to global frame start + j.  Nothing is exchanged.
    """
    info = info or rank_info()
    start, stop = shard_range(len(frames), info.world, info.rank)
    results = []
    for s in range(start, stop, batch):
        results.extend(process_batch(frames[s:min(stop, s + batch)]))
    if len(results) != stop - start:
        raise RuntimeError(f"process_batch returned {len(results)} results for "
                           f"{stop - start} frames")
    return start, stop, results


def gather_shards(start: int, results: list) -> list:
    """Bookkeeping only (never on the timed data path): every rank's (start, results)
    gathered to all ranks and placed at their global frame offsets."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(results)
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, (start, list(results)))
    n = sum(len(r) for _, r in parts)
    out = [None] * n
    for s, r in parts:
        out[s:s + len(r)] = r
    return out


class MultiDevicePipeline:
    """One process driving several GPUs: a HostPipeline (own streams, pinned buffers and
    CUDA graphs) and one host thread per device; a host batch is split into contiguous
    per-device shards (shard_range), with no collective and no cross-device traffic.

    run(src_host) -> list of per-device FrontEndResult, in frame order, each covering
    its shard ([start, stop) in `self.shards`).  The same device may appear twice (two
    independent pipelines on one GPU, e.g. to test the driver on a one-GPU box).
    """

    def __init__(self, M, N, devices=None, **pipeline_kwargs):
        from .frontend import HostPipeline
        if devices is None:
            devices = list(range(torch.cuda.device_count()))
        self.devices = [torch.device("cuda", d) if isinstance(d, int) else torch.device(d)
                        for d in devices]
        if not self.devices:
            raise RuntimeError("MultiDevicePipeline: no CUDA device")
        self.pipes = []
        for d in self.devices:
            with torch.cuda.device(d):
                self.pipes.append(HostPipeline(M, N, device=d, **pipeline_kwargs))
        self.shards = []

    def run(self, src_host: torch.Tensor):
        import threading
        F = src_host.shape[0]
        n = len(self.pipes)
        self.shards = [shard_range(F, n, r) for r in range(n)]
        results = [None] * n
        errors = []

        def work(r):
            a, b = self.shards[r]
            try:
                with torch.cuda.device(self.devices[r]):
                    if b > a:
                        results[r] = self.pipes[r].run(src_host[a:b])
            except BaseException as e:  # noqa: BLE001 - re-raised on the caller's thread
                errors.append(e)

        threads = [threading.Thread(target=work, args=(r,)) for r in range(n)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
        self.h2d_bytes = sum(getattr(p, "h2d_bytes", 0) for p, r in zip(self.pipes, results) if r)
        self.d2h_bytes = sum(getattr(p, "d2h_bytes", 0) for p, r in zip(self.pipes, results) if r)
        return results
