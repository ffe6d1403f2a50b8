"""Stream sharding across GPUs (one process per GPU, torch.distributed).

The streams of a batched configuration are independent solvers,
so a job of B streams is split over G ranks in contiguous blocks of B/G by
global stream index -- no collective touches the hot path.  Inputs are keyed by
the global index (workloads.device_batch), so every stream's bytes and results
are identical for any G.  The only communication is outside the timed region:
the max-over-ranks of the step time, and an optional gather of per-stream
rank/status vectors (a few bytes per stream).
"""

from __future__ import annotations


def shard_range(num_streams: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [b0, b1) of global stream indices owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    if num_streams % world:
        raise ValueError(f"{num_streams} streams do not shard evenly over {world} ranks")
    per = num_streams // world
    return rank * per, (rank + 1) * per


def _dev(device):
    """Collectives run on the device for NCCL and on the host for gloo."""
    import torch.distributed as dist

    return None if dist.get_backend() == "gloo" else device


def max_over_ranks(value: float, device=None) -> float:
    """Max of a float over all ranks (identity without a process group)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_dev(device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_dev(device))
    dist.all_reduce(t)
    return float(t.item())


def gather_streams(local, device=None):
    """All-gather a per-stream vector (rank, status, ...) in global stream order."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    local = local.to(_dev(device) or "cpu")
    parts = [torch.empty_like(local) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, local.contiguous())
    return torch.cat(parts)
