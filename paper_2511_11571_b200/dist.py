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
    tensor on every rank (verification only). NCCL needs CUDA tensors, gloo
    CPU tensors: pass `local` on the backend's device."""
    world = dist.get_world_size(group)
    sizes = [shard_range(n_units, world, r) for r in range(world)]
    maxh = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((maxh, *local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[: hi - lo] for p, (lo, hi) in zip(parts, sizes)], dim=0)


def shard_fwd_bwd(q, k, v, dout, block_size: int, top_k: int, rank: int, world: int, *, mode: str = "tc",
                  deterministic: bool = False):
    """This rank's part of a fixed global head set: heads [lo, hi) of the
    [H, N, d] bf16 CUDA inputs through moba_attn forward + backward, with no
    communication. Returns ((lo, hi), out, lse, dq, dk, dv)."""
    from .attention import moba_attn
    lo, hi = shard_range(q.shape[0], world, rank)
    xs = [t[lo:hi].detach().clone().requires_grad_(True) for t in (q, k, v)]
    out, lse = moba_attn(*xs, block_size, top_k, mode=mode, deterministic=deterministic, return_lse=True)
    out.backward(dout[lo:hi])
    return (lo, hi), out.detach(), lse.detach(), xs[0].grad, xs[1].grad, xs[2].grad


def gather_and_compare(local: dict, reference: dict | None, n_heads: int, device, group=None) -> dict:
    """Gather every rank's result tensors (name -> [h_r, ...]) to all ranks;
    when `reference` (name -> full [n_heads, ...] tensor, rank 0's
    single-GPU run) is given, return per-name (bitwise_equal, max_abs_diff)."""
    out = {}
    for name, t in local.items():
        full = gather_heads(t.to(device), n_heads, group=group)
        if reference is not None:
            ref = reference[name].to(full.device)
            diff = float((full.float() - ref.float()).abs().max()) if full.numel() else 0.0
            out[name] = (bool(torch.equal(full, ref)), diff)
    return out
