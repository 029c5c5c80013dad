"""Configuration, errors, counters and the device routing plan.

Mirrors the reference's core types (src/core.py) so callers switch by
changing the import: `MobaConfig` (src/core.py:155-190), `OpCounters`
(src/core.py:193-226), `RoutingPlan` (src/core.py:229-251), the `MobaError`
hierarchy (src/core.py:17-38) and `resolve_threads` (src/core.py:299-314).

Differences, by design:
  * a RoutingPlan lives on the GPU (int32 CUDA tensors for any number of
    heads); its reference-named attributes (`topk_indices`, `counts`,
    `offsets`, `flat_queries`) read back numpy arrays (int32 / int64 /
    int64 / int32 like the reference) and accept assignment, which uploads;
  * the plan additionally carries `row_pos`, the (query, slot) -> flat
    position inverse map the combine kernel uses.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np


class MobaError(Exception):
    """Base class for all package errors (src/core.py:17-18)."""


class FormatError(MobaError):
    """Malformed tensor file header (src/core.py:21-22)."""


class LengthError(MobaError):
    """Tensor file payload length mismatch (src/core.py:25-26)."""


class ShapeError(MobaError):
    """Array shape or dtype violates an operation's precondition (src/core.py:29-30)."""


class ConfigError(MobaError):
    """Invalid MobaConfig or parameters (src/core.py:33-34)."""


class PlanValidationError(MobaError):
    """RoutingPlan is inconsistent or violates causality (src/core.py:37-38)."""


@dataclass(frozen=True)
class MobaConfig:
    """Block size, top-k, head dim and tiling knobs (src/core.py:155-190).

    top_k counts the routed PAST blocks; the own block is always attended in
    addition, so index rows carry top_k + 1 entries (src/core.py:160-162).
    The logical/physical tile fields are accepted for signature parity; the
    GPU kernels use their own compile-time tiles (results are
    tile-invariant, tests/test_router.py:77-89).
    """

    block_size_B: int
    top_k: int
    head_dim_d: int
    logical_q_block_Bq: int = 512
    phys_tile_Br: int | None = None
    phys_tile_Bc: int | None = None
    conv_width: int = 0

    def __post_init__(self):
        if self.block_size_B < 1 or self.top_k < 1 or self.head_dim_d < 1:
            raise ConfigError("block_size_B, top_k, head_dim_d must all be >= 1")
        if self.logical_q_block_Bq < 1:
            raise ConfigError("logical_q_block_Bq must be >= 1")
        if self.phys_tile_Br is None:
            object.__setattr__(self, "phys_tile_Br", min(64, self.logical_q_block_Bq))
        if self.phys_tile_Bc is None:
            object.__setattr__(self, "phys_tile_Bc", min(64, self.block_size_B))
        if not 1 <= self.phys_tile_Bc <= self.block_size_B:
            raise ConfigError(f"phys_tile_Bc={self.phys_tile_Bc} must be in [1, block_size_B]")
        if not 1 <= self.phys_tile_Br <= self.logical_q_block_Bq:
            raise ConfigError(f"phys_tile_Br={self.phys_tile_Br} must be in [1, logical_q_block_Bq]")
        if self.conv_width not in (0, 3, 5):
            raise ConfigError(f"conv_width must be 0, 3, or 5, got {self.conv_width}")

    def n_blocks(self, n_tokens: int) -> int:
        return -(-n_tokens // self.block_size_B)


@dataclass
class OpCounters:
    """Operation counters (src/core.py:193-226).

    On the GPU path the counters are filled from the plan in closed form
    with the reference's tile knobs and classification rules
    (paper_2511_11571_b200/counters.py): the same four numbers the
    reference's tile walk produces (checked against reference-generated
    values, tests/golden/counters.npz).
    """

    score_flops: int = 0
    attn_flops: int = 0
    gathered_elems: int = 0
    bulk_elems: int = 0

    def reset(self) -> None:
        self.score_flops = self.attn_flops = self.gathered_elems = self.bulk_elems = 0

    def merge(self, other: "OpCounters") -> None:
        self.score_flops += other.score_flops
        self.attn_flops += other.attn_flops
        self.gathered_elems += other.gathered_elems
        self.bulk_elems += other.bulk_elems

    def as_dict(self) -> dict:
        return {
            "score_flops": self.score_flops,
            "attn_flops": self.attn_flops,
            "gathered_elems": self.gathered_elems,
            "bulk_elems": self.bulk_elems,
        }


def resolve_threads(requested: int | None = None) -> int:
    """Worker count capped by MOBA_THREADS (src/core.py:299-314). Kept for
    signature parity: GPU work is not split over host threads."""
    cap = os.environ.get("MOBA_THREADS", "0")
    try:
        cap_val = int(cap)
    except ValueError:
        cap_val = 0
    if cap_val <= 0:
        cap_val = min(4, os.cpu_count() or 1)
    if requested is None or requested <= 0:
        requested = cap_val
    return max(1, min(requested, cap_val))


class RoutingPlan:
    """Query-centric top-k selection plus its key-block-major varlen layout,
    resident on the GPU (src/core.py:229-251).

    Device fields (int32 CUDA tensors):
      topk     [H, N, width]   ascending block ids, -1 tail
      counts_d [H, n]          queries per block
      offsets_d[H, n]          exclusive prefix sum (head-local)
      flat_d   [H, N*width]    block-major query lists; head h's valid
                               region is flat_d[h, :counts_d[h].sum()]
      row_pos  [H, N, width]   flat position of (query, slot), -1 sentinel
    The reference attribute names return host numpy copies; for H == 1 the
    head dimension is dropped, matching the reference's per-head plan.
    """

    def __init__(self, topk, counts, offsets, flat, row_pos, n_tokens: int, block_size: int):
        self.topk = topk
        self.counts_d = counts
        self.offsets_d = offsets
        self.flat_d = flat
        self.row_pos = row_pos
        self.n_tokens = int(n_tokens)
        self.block_size = int(block_size)
        self._row_pos_stale = row_pos is None

    # -- shape helpers -------------------------------------------------
    @property
    def n_heads(self) -> int:
        return int(self.topk.shape[0])

    @property
    def width(self) -> int:
        return int(self.topk.shape[2])

    @property
    def n_blocks(self) -> int:
        return int(self.counts_d.shape[1])

    @property
    def n_queries(self) -> int:
        return self.n_tokens

    def _squeeze(self, a):
        return a[0] if self.n_heads == 1 else a

    # -- reference-named host views (src/core.py:243-251) -------------
    @property
    def topk_indices(self) -> np.ndarray:
        return self._squeeze(self.topk.cpu().numpy().astype(np.int32))

    @topk_indices.setter
    def topk_indices(self, value):
        self.topk = _upload_i32(value, self.topk)
        self._row_pos_stale = True

    @property
    def counts(self) -> np.ndarray:
        return self._squeeze(self.counts_d.cpu().numpy().astype(np.int64))

    @counts.setter
    def counts(self, value):
        self.counts_d = _upload_i32(value, self.counts_d)
        self._row_pos_stale = True

    @property
    def offsets(self) -> np.ndarray:
        return self._squeeze(self.offsets_d.cpu().numpy().astype(np.int64))

    @offsets.setter
    def offsets(self, value):
        self.offsets_d = _upload_i32(value, self.offsets_d)
        self._row_pos_stale = True

    @property
    def flat_queries(self) -> np.ndarray:
        tot = self.counts_d.sum(dim=1).cpu().numpy()
        f = self.flat_d.cpu().numpy()
        rows = [f[h, : int(tot[h])].astype(np.int32) for h in range(self.n_heads)]
        return rows[0] if self.n_heads == 1 else rows

    @flat_queries.setter
    def flat_queries(self, value):
        import torch
        vals = [value] if self.n_heads == 1 else list(value)
        cap = self.flat_d.shape[1]
        out = torch.zeros_like(self.flat_d)
        for h, v in enumerate(vals):
            v = np.asarray(v, dtype=np.int64)
            if v.size > cap:
                raise PlanValidationError("flat_queries longer than N * width")
            out[h, : v.size] = torch.as_tensor(v.astype(np.int32))
        self.flat_d = out
        self._row_pos_stale = True

    def head(self, h: int) -> "RoutingPlan":
        """Single-head view (device tensors are sliced, not copied)."""
        sl = slice(h, h + 1)
        # a stale inverse map (a field was reassigned) is not handed down:
        # the child rebuilds it from its own fields when it needs it
        rp = None if (self.row_pos is None or self._row_pos_stale) else self.row_pos[sl]
        return RoutingPlan(self.topk[sl], self.counts_d[sl], self.offsets_d[sl], self.flat_d[sl], rp,
                           self.n_tokens, self.block_size)


def _upload_i32(value, like):
    import torch
    t = torch.as_tensor(np.asarray(value).astype(np.int64))
    if t.dim() == like.dim() - 1:
        t = t.unsqueeze(0)
    if tuple(t.shape) != tuple(like.shape):
        raise PlanValidationError(f"plan field shape {tuple(t.shape)} does not match {tuple(like.shape)}")
    if t.numel() and (int(t.max()) > 2**31 - 1 or int(t.min()) < -2**31):
        raise PlanValidationError("plan field out of int32 range")
    return t.to(device=like.device, dtype=torch.int32).contiguous()
