"""Batch x heads sharding over GPUs (one process per GPU).

MoBA heads are independent (the reference loops heads at
src/cli.py:259-281), so the hot path shards by contiguous (batch, head)
ranges with NO collective on the data path. A collective appears only to
gather outputs for verification (all_gather over NCCL on GPUs, gloo on CPU).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_units: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) of n_units for `rank`; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    base, extra = divmod(n_units, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_heads(local: torch.Tensor, n_units: int, group=None) -> torch.Tensor:
    """All-gather per-rank head shards [h_r, ...] into the full [n_units, ...]
    tensor on every rank (verification only)."""
    world = dist.get_world_size(group)
    sizes = [shard_range(n_units, world, r) for r in range(world)]
    maxh = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((maxh, *local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[: hi - lo] for p, (lo, hi) in zip(parts, sizes)], dim=0)
