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
    if dev is None:
        dev = torch.device("cuda", torch.cuda.current_device()) \
            if dist.get_backend() == "nccl" else torch.device("cpu")
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
    front end on a (<= batch, M, N, 3) slice and returns per-frame triangle counts.
    Returns (start, stop, per-frame counts) for this rank; nothing is exchanged.
    """
    info = info or rank_info()
    start, stop = shard_range(len(frames), info.world, info.rank)
    counts = []
    for s in range(start, stop, batch):
        counts.extend(process_batch(frames[s:min(stop, s + batch)]))
    return start, stop, counts
