"""Routing pipeline — centroids, tiled top-k, varlen plan — on the GPU.

Drop-in for the reference's router module (src/router.py): same names,
argument meaning and errors. Numpy in -> numpy out (plan fields read back
on demand); torch CUDA in -> torch CUDA out.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib
from .counters import add_plan_counters
from ._convert import routing_heads, to_heads
from .core import MobaConfig, OpCounters, PlanValidationError, RoutingPlan, ShapeError

ROUTE_MODES = {"fp32": _lib.MOBA_ROUTE_FP32, "tc": _lib.MOBA_ROUTE_TC}


@dataclass
class CentroidMatrix:
    """Block centroids plus per-block token counts (src/router.py:20-29).

    `device` holds the fp32 [H, n, Dp] kernel-layout centroids; `centroids`
    is the caller-layout view (numpy [n, d] for numpy callers)."""

    centroids: object
    block_lengths: np.ndarray
    device: torch.Tensor = None
    block_size: int = 0

    @property
    def n_blocks(self) -> int:
        return int(self.block_lengths.shape[0])


def _lengths(N: int, B: int) -> np.ndarray:
    n = -(-N // B)
    return np.minimum(B, N - np.arange(n) * B).astype(np.int64)


def compute_centroids(K, B: int, counters: OpCounters | None = None) -> CentroidMatrix:
    """Mean of each block of B key rows, ragged last block (src/router.py:32-46)."""
    if B < 1:
        raise ShapeError("block size must be >= 1")
    if (isinstance(K, np.ndarray) and K.ndim != 2):
        raise ShapeError("K must be 2-D (N x d)")
    k, info = to_heads(K, "K")
    k32 = routing_heads(K, "K", device=k.device)
    cent, _ = _device.centroids(k if k32 is None else k32, B)
    if counters is not None:    # src/router.py:44-45
        counters.bulk_elems += k.shape[0] * (info.n_tokens * info.d + cent.shape[1] * info.d)
    view = cent[..., : info.d]
    if info.kind == "numpy":
        view = view.reshape(*info.lead, cent.shape[1], info.d).cpu().numpy().astype(info.np_dtype)
    else:
        view = view.reshape(*info.lead, cent.shape[1], info.d)
    return CentroidMatrix(view, _lengths(info.n_tokens, B), cent, B)


def _route(Q, cents: CentroidMatrix, cfg: MobaConfig, counters, mode: str) -> tuple[RoutingPlan, object]:
    if isinstance(Q, np.ndarray) and Q.ndim != 2:
        raise ShapeError("Q must be 2-D (N x d)")
    q, info = to_heads(Q, "Q")
    cent = cents.device
    if cent is None or cents.block_size != cfg.block_size_B:
        raise ShapeError("centroids were not computed by this package for block_size_B")
    if cent.shape[0] != q.shape[0] or cent.shape[2] != q.shape[2]:
        raise ShapeError(f"centroid layout {tuple(cent.shape)} does not match Q {tuple(q.shape)}")
    q32 = routing_heads(Q, "Q", device=q.device) if mode == "fp32" else None
    plan = _device.route(q if q32 is None else q32, cent, cfg.block_size_B, cfg.top_k, ROUTE_MODES[mode])
    if counters is not None:    # select_topk only (src/router.py:85-88); the centroids were counted above
        c = type(counters)()
        add_plan_counters(c, q.shape[0], info.n_tokens, info.d, cfg.block_size_B, cfg.phys_tile_Br)
        counters.score_flops += c.score_flops
        counters.bulk_elems += c.bulk_elems - q.shape[0] * (info.n_tokens * info.d + cent.shape[1] * info.d)
    return plan, info


def select_topk(Q, centroids: CentroidMatrix, cfg: MobaConfig,
                counters: OpCounters | None = None, mode: str = "fp32"):
    """N x (top_k + 1) index matrix: own block plus the top_k strictly-past
    blocks by unscaled q . centroid, ties to the lower index, rows ascending,
    -1 tail (src/router.py:49-120)."""
    plan, info = _route(Q, centroids, cfg, counters, mode)
    if info.kind == "numpy":
        return plan.topk_indices
    return plan.topk.reshape(*info.lead, info.n_tokens, cfg.top_k + 1)


def build_varlen(topk_indices, n_blocks: int) -> RoutingPlan:
    """Key-block-major varlen layout from an index matrix (src/router.py:123-154).

    The block size is recovered from (N, n_blocks) as the reference's plans
    only ever use B with ceil(N / B) == n_blocks; pass a RoutingPlan-producing
    call (build_plan) when B is ambiguous.
    """
    if isinstance(topk_indices, torch.Tensor):
        idx = topk_indices
        if idx.dim() == 2:
            idx = idx.unsqueeze(0)
        if idx.dim() != 3:
            raise ShapeError("topk_indices must be 2-D (or [H, N, width])")
        idx = idx.to(torch.device("cuda", torch.cuda.current_device()) if not idx.is_cuda else idx.device)
        N = idx.shape[1]
        if idx.numel():
            lo, hi = int(idx.min()), int(idx.max())
            if lo < -1 or hi >= n_blocks:
                raise PlanValidationError(f"index entries must lie in [-1, {n_blocks}), got [{lo}, {hi}]")
    else:
        arr = np.asarray(topk_indices)
        if arr.ndim != 2:
            raise ShapeError("topk_indices must be 2-D")
        if arr.size and (arr.min() < -1 or arr.max() >= n_blocks):
            raise PlanValidationError(
                f"index entries must lie in [-1, {n_blocks}), got [{int(arr.min())}, {int(arr.max())}]")
        N = arr.shape[0]
        idx = torch.as_tensor(arr.astype(np.int32)).unsqueeze(0).cuda()
    B = infer_block_size(N, n_blocks)
    return _device.varlen(idx.to(torch.int32).contiguous(), B)


def infer_block_size(N: int, n_blocks: int) -> int:
    """Smallest B with ceil(N / B) == n_blocks (the reference's plans satisfy it)."""
    if n_blocks < 1:
        raise PlanValidationError("n_blocks must be >= 1")
    B = -(-N // n_blocks)
    if -(-N // B) != n_blocks:
        raise PlanValidationError(f"no block size gives {n_blocks} blocks for N={N}")
    return B


def build_plan(Q, K, cfg: MobaConfig, counters: OpCounters | None = None, mode: str = "fp32") -> RoutingPlan:
    """centroids -> tiled top-k -> varlen (src/router.py:157-161)."""
    cents = compute_centroids(K, cfg.block_size_B, counters)
    plan, _ = _route(Q, cents, cfg, counters, mode)
    return plan
