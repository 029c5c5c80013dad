"""OpCounters of the reference in closed form, computed from a routing plan.

The reference counts multiply-adds and element traffic while it walks its
tiles (src/core.py:193-226). The GPU kernels tile differently, so the same
numbers are derived here from the plan and the reference's tile knobs
(MobaConfig.logical_q_block_Bq / phys_tile_Br, src/core.py:168-181), with
the reference's classification rules:

  compute_centroids   bulk += N*d + n*d                     (src/router.py:44-45)
  select_topk         per Br-row tile [r0, r1) with L = min(n, (r1-1)//B):
                      score += (r1-r0)*L*d, bulk += L*d     (src/router.py:85-88)
  moba_forward        per (Bq query block, key block j) the attending
                      queries in Br-row tiles; each tile moves n*(3d+4)
                      elements (gather Q, gather + scatter (m, l, acc)) —
                      bulk when its query ids are one contiguous run, else
                      gathered (_move, src/attention.py:77-86) — and loads
                      K_j, V_j (2*len_j*d bulk); attn += 2d per visible pair;
                      final O / L writes bulk += N*(d+1)   (src/attention.py:96-144)
  moba_backward       bulk += 2Nd + N (D); per key block with queries: K_j,
                      V_j loads and dK_j, dV_j writes (4*len_j*d bulk); its
                      slice in Br-row tiles moving n*(2d+2) elements
                      (bulk / gathered as above); attn += 5d per visible
                      pair; dQ write bulk += N*d           (src/attention.py:204-300)

Everything is vectorised torch on the plan's own device (CPU tensors work
too); it runs only when the caller passes an OpCounters object.
"""

from __future__ import annotations

import torch


def _block_lengths(n_tokens: int, block_size: int, n_blocks: int, device) -> torch.Tensor:
    j = torch.arange(n_blocks, device=device, dtype=torch.int64)
    return torch.clamp(n_tokens - j * block_size, max=block_size)


def _entries(counts_h: torch.Tensor, flat_h: torch.Tensor):
    """(block id, query id) of every plan entry of one head, block-major."""
    counts_h = counts_h.to(torch.int64)
    total = int(counts_h.sum())
    blk = torch.repeat_interleave(torch.arange(counts_h.numel(), device=counts_h.device), counts_h)
    return blk, flat_h[:total].to(torch.int64)


def _tile_traffic(group: torch.Tensor, q: torch.Tensor, tile_rows: int, elems_per_row: int) -> tuple[int, int]:
    """Split the runs of equal `group` (contiguous in entry order) into
    tiles of tile_rows entries; return (bulk, gathered) element counts with
    a tile counted bulk when its query ids form one contiguous run."""
    E = group.numel()
    if E == 0:
        return 0, 0
    idx = torch.arange(E, device=group.device)
    start = torch.ones(E, dtype=torch.bool, device=group.device)
    start[1:] = group[1:] != group[:-1]
    first = torch.cummax(torch.where(start, idx, torch.zeros_like(idx)), dim=0).values
    rank = idx - first
    tile_start = rank % tile_rows == 0
    tile_id = torch.cumsum(tile_start.to(torch.int64), dim=0) - 1
    n_tiles = int(tile_id[-1]) + 1
    size = torch.zeros(n_tiles, dtype=torch.int64, device=group.device).index_add_(0, tile_id, torch.ones_like(idx))
    q_first = q[tile_start]
    tile_end = torch.ones(E, dtype=torch.bool, device=group.device)
    tile_end[:-1] = tile_id[1:] != tile_id[:-1]
    q_last = q[tile_end]
    contiguous = (size == 1) | (q_last - q_first + 1 == size)
    elems = size * elems_per_row
    return int(elems[contiguous].sum()), int(elems[~contiguous].sum())


def add_plan_counters(counters, n_heads: int, n_tokens: int, d: int, block_size: int, tile_rows: int) -> None:
    """compute_centroids + select_topk counters of n_heads heads (they
    depend on N, d, B and Br only, not on the data)."""
    N, B = n_tokens, block_size
    n = -(-N // B)
    r0 = torch.arange(0, N, tile_rows, dtype=torch.int64)
    r1 = torch.clamp(r0 + tile_rows, max=N)
    L = torch.clamp((r1 - 1) // B, max=n)
    counters.score_flops += n_heads * int(((r1 - r0) * L).sum()) * d
    counters.bulk_elems += n_heads * (N * d + n * d + int(L.sum()) * d)


def add_forward_counters(counters, plan, d: int, cfg, visible: int) -> None:
    N, B = plan.n_tokens, plan.block_size
    lens = _block_lengths(N, B, plan.n_blocks, plan.counts_d.device)
    nq = -(-N // cfg.logical_q_block_Bq)
    bulk = gathered = 0
    for h in range(plan.n_heads):
        blk, q = _entries(plan.counts_d[h], plan.flat_d[h])
        group = blk * nq + q // cfg.logical_q_block_Bq
        b, g = _tile_traffic(group, q, cfg.phys_tile_Br, 3 * d + 4)
        bulk += b
        gathered += g
        # K_j, V_j per tile: tiles of block j = sum over its query blocks of ceil(m / Br)
        if group.numel():
            gs = torch.unique_consecutive(group, return_counts=True)
            gblk = gs[0] // nq
            tiles = (gs[1] + cfg.phys_tile_Br - 1) // cfg.phys_tile_Br
            bulk += int((tiles * 2 * lens[gblk] * d).sum())
        bulk += N * (d + 1)
    counters.attn_flops += 2 * d * visible
    counters.bulk_elems += bulk
    counters.gathered_elems += gathered


def add_backward_counters(counters, plan, d: int, cfg, visible: int) -> None:
    N, B = plan.n_tokens, plan.block_size
    lens = _block_lengths(N, B, plan.n_blocks, plan.counts_d.device)
    bulk = gathered = 0
    for h in range(plan.n_heads):
        blk, q = _entries(plan.counts_d[h], plan.flat_d[h])
        b, g = _tile_traffic(blk, q, cfg.phys_tile_Br, 2 * d + 2)
        bulk += b
        gathered += g
        nonempty = plan.counts_d[h] > 0
        bulk += 2 * N * d + N + int((4 * lens[nonempty] * d).sum()) + N * d
    counters.attn_flops += 5 * d * visible
    counters.bulk_elems += bulk
    counters.gathered_elems += gathered
