"""Frame sharding across ranks: frames are independent, so
rank r of N takes a contiguous frame range and no data-path collective exists.
The only collective is the untimed max-over-ranks of the measured times."""

from __future__ import annotations

import os


def env_rank_world() -> tuple[int, int, int]:
    """(rank, local_rank, world_size) from the torchrun environment."""
    return int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))


def frame_range(rank: int, world: int, total: int | None = None, per_rank: int | None = None) -> tuple[int, int]:
    """[start, stop) of this rank's frames.

    ``per_rank`` (weak scaling: fixed frames per GPU) or ``total`` (strong
    scaling: a fixed batch split as evenly as possible, e.g. BASELINE config 3's
    8192 frames over 1/2/4/8 GPUs)."""
    if per_rank is not None:
        return rank * per_rank, (rank + 1) * per_rank
    if total is None:
        raise ValueError("give total or per_rank")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def max_over_ranks(values, device=None):
    """Element-wise max of a list of floats over all ranks (no-op when not distributed)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]
