"""Multi-GPU layout of the hot path: independent camera streams are partitioned
across GPUs, one backbone+heads replica per GPU, with NO collective on the data path.
torch.distributed only provides the start barrier and the max-over-ranks of the timed region.
"""

from __future__ import annotations


def streams_for_rank(n_streams: int, rank: int, world: int) -> list[int]:
    """Camera stream i runs on GPU i mod world (SURVEY §8e partitioning)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    return [i for i in range(n_streams) if i % world == rank]


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """The job's wall time is the slowest rank's device time."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def total_frames(per_rank_frames: int, dist=None, device=None) -> int:
    if dist is None or not dist.is_initialized():
        return per_rank_frames
    import torch
    t = torch.tensor([per_rank_frames], dtype=torch.int64, device=device)
    dist.all_reduce(t)
    return int(t.item())
