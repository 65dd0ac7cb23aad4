"""Multi-GPU plumbing: shard TX positions across ranks, gather outputs to root.

SURVEY.md section 8(e): positions are independent units, so a batch of B
positions is split contiguously across P ranks (one process per GPU), the
scene and MLP weights are replicated on every GPU, and the only collective is
the final gather of the rendered outputs to rank 0 (NCCL over NVLink on the
GPUs; the same code runs on gloo for the CPU tests). Nothing here computes a
spectrum: rendering is libswr.so's job on each rank's own device.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, start + count) share of `total` units for `rank`;
    the first total % world ranks take one extra unit."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def gather_to_root(local: torch.Tensor, total: int, world: int, rank: int, root: int = 0):
    """Gather the ranks' contiguous shards (dim 0) into one tensor on `root`.
    Shards may differ by one row (shard_range); they are padded to a common
    length for the collective and trimmed afterwards. Returns the full tensor
    on root and None elsewhere."""
    if world == 1:
        return local
    per = -(-total // world)
    start, count = shard_range(total, world, rank)
    if local.shape[0] != count:
        raise ValueError("local shard has the wrong length")
    pad = local
    if count < per:
        pad = torch.zeros((per,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        pad[:count] = local
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == root else None
    dist.gather(pad, gather_list=bufs, dst=root)
    if rank != root:
        return None
    parts = []
    for r in range(world):
        _, c = shard_range(total, world, r)
        parts.append(bufs[r][:c])
    return torch.cat(parts, dim=0)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
