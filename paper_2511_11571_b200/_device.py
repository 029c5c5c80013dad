"""Thin device-level wrappers over the C ABI.

Every function takes/returns CUDA tensors in the kernel layout: bf16
[H, N, Dp] with Dp in {64, 128} (channels zero-padded), int32 plan arrays,
fp32 centroids / LSE. No computation happens here beyond allocation; a
missing library or device raises (no CPU fallback).
"""

from __future__ import annotations

import math

import torch

from . import _lib
from .core import ConfigError, PlanValidationError, RoutingPlan, ShapeError

SUPPORTED_DP = (64, 128)
MAX_TOP_K = 31
MAX_BLOCK = 512


def padded_dim(d: int) -> int:
    for dp in SUPPORTED_DP:
        if d <= dp:
            return dp
    raise ConfigError(f"head_dim {d} > 128 is not supported by the compiled kernels")


def require_cuda(t: torch.Tensor, name: str) -> None:
    if not t.is_cuda:
        raise ShapeError(f"{name} must be a CUDA tensor")


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def centroids(k: torch.Tensor, block_size: int, conv_w: torch.Tensor | None = None):
    """(centroids fp32 [H, n, Dp], k_used bf16 [H, N, Dp]); k_used is the
    conv output when conv_w is given, else k itself. An fp32 `k` (numpy f32 /
    f64 callers) is pooled unrounded; its k_used is the bf16 copy (or the
    bf16 K' of the conv)."""
    lib = _lib.load()
    H, N, Dp = k.shape
    n = -(-N // block_size)
    cent = torch.empty((H, n, Dp), dtype=torch.float32, device=k.device)
    k_out = None
    width = 0
    if conv_w is not None:
        width = int(conv_w.shape[0])
        conv_w = conv_w.to(device=k.device, dtype=torch.float32).contiguous()
        k_out = torch.empty((H, N, Dp), dtype=torch.bfloat16, device=k.device)
    fn = lib.moba_centroids_f32 if k.dtype == torch.float32 else lib.moba_centroids
    st = fn(k.data_ptr(), _lib.ptr(conv_w), width, H, N, Dp, block_size, _lib.ptr(k_out), cent.data_ptr(), _stream(k))
    _lib.check(st, "moba_centroids")
    if k_out is not None:
        return cent, k_out
    return cent, (k.to(torch.bfloat16) if k.dtype != torch.bfloat16 else k)


def _empty_plan(H, N, width, n, device):
    i32 = dict(dtype=torch.int32, device=device)
    return (torch.empty((H, N, width), **i32), torch.empty((H, n), **i32), torch.empty((H, n), **i32),
            torch.empty((H, N * width), **i32), torch.empty((H, N, width), **i32))


def kv_group_of(q: torch.Tensor, kv: torch.Tensor) -> int:
    """Query heads per K/V head (GQA/MQA; 1 = MHA)."""
    Hq, Hk = q.shape[0], kv.shape[0]
    if Hk < 1 or Hq % Hk != 0:
        raise ShapeError(f"{Hq} query heads are not a multiple of {Hk} key/value heads")
    return Hq // Hk


def route(q: torch.Tensor, cent: torch.Tensor, block_size: int, top_k: int, mode: int = _lib.MOBA_ROUTE_FP32):
    """Routing plan per QUERY head; `cent` may have fewer (K/V) heads (GQA:
    query head h routes against the centroids of K/V head h // group)."""
    lib = _lib.load()
    H, N, Dp = q.shape
    G = kv_group_of(q, cent)
    if top_k > MAX_TOP_K:
        raise ConfigError(f"top_k={top_k} > {MAX_TOP_K} is not supported by the compiled kernels")
    n = cent.shape[1]
    width = top_k + 1
    topk, counts, offsets, flat, row_pos = _empty_plan(H, N, width, n, q.device)
    ws = _ws(lib.moba_route_workspace_size(H, N, block_size, top_k), q.device)
    if q.dtype == torch.float32 and mode == _lib.MOBA_ROUTE_FP32:
        # numpy f32 / f64 callers: route on the unrounded queries
        st = lib.moba_route_f32(q.data_ptr(), cent.data_ptr(), H, G, N, Dp, block_size, top_k,
                                topk.data_ptr(), counts.data_ptr(), offsets.data_ptr(), flat.data_ptr(),
                                row_pos.data_ptr(), ws.data_ptr(), ws.numel(), _stream(q))
    else:
        qb = q if q.dtype == torch.bfloat16 else q.to(torch.bfloat16)
        st = lib.moba_route_gqa(qb.data_ptr(), cent.data_ptr(), H, G, N, Dp, block_size, top_k, mode,
                                topk.data_ptr(), counts.data_ptr(), offsets.data_ptr(), flat.data_ptr(),
                                row_pos.data_ptr(), ws.data_ptr(), ws.numel(), _stream(q))
    _lib.check(st, "moba_route")
    return RoutingPlan(topk, counts, offsets, flat, row_pos, N, block_size)


def varlen(topk: torch.Tensor, block_size: int) -> RoutingPlan:
    lib = _lib.load()
    H, N, width = topk.shape
    if width > 32:
        raise ConfigError("index rows wider than 32 are not supported by the compiled kernels")
    n = -(-N // block_size)
    topk = topk.to(torch.int32).contiguous()
    _, counts, offsets, flat, row_pos = _empty_plan(H, N, width, n, topk.device)
    ws = _ws(lib.moba_route_workspace_size(H, N, block_size, width - 1), topk.device)
    st = lib.moba_varlen(topk.data_ptr(), H, N, width, block_size, counts.data_ptr(), offsets.data_ptr(),
                         flat.data_ptr(), row_pos.data_ptr(), ws.data_ptr(), ws.numel(), _stream(topk))
    _lib.check(st, "moba_varlen")
    return RoutingPlan(topk, counts, offsets, flat, row_pos, N, block_size)


def validate(plan: RoutingPlan, n_tokens: int, block_size: int) -> None:
    """validate_plan (src/core.py:254-296): shapes here, invariants on device."""
    lib = _lib.load()
    n = -(-n_tokens // block_size)
    H = plan.n_heads
    if plan.topk.dim() != 3 or plan.topk.shape[1] != n_tokens:
        raise PlanValidationError(f"topk_indices shape {tuple(plan.topk.shape)} does not match N={n_tokens}")
    if tuple(plan.counts_d.shape) != (H, n) or tuple(plan.offsets_d.shape) != (H, n):
        raise PlanValidationError("counts/offsets length does not match the block count")
    if plan.flat_d.shape[1] != n_tokens * plan.width:
        raise PlanValidationError("flat_queries capacity does not match N * width")
    ws = _ws(256 + 8 * H, plan.topk.device)
    st = lib.moba_validate_plan(plan.topk.data_ptr(), plan.counts_d.data_ptr(), plan.offsets_d.data_ptr(),
                                plan.flat_d.data_ptr(), H, n_tokens, plan.width, block_size,
                                ws.data_ptr(), ws.numel(), _stream(plan.topk))
    _lib.check(st, "validate_plan")


def ensure_row_pos(plan: RoutingPlan) -> None:
    if plan.row_pos is not None and not plan._row_pos_stale:
        return
    lib = _lib.load()
    H, N, width = plan.topk.shape
    rp = torch.empty((H, N, width), dtype=torch.int32, device=plan.topk.device)
    st = lib.moba_plan_row_pos(plan.topk.data_ptr(), plan.counts_d.data_ptr(), plan.offsets_d.data_ptr(),
                               plan.flat_d.data_ptr(), H, N, width, plan.block_size, rp.data_ptr(),
                               _stream(plan.topk))
    _lib.check(st, "moba_plan_row_pos")
    plan.row_pos = rp
    plan._row_pos_stale = False


def fwd(q, k, v, plan: RoutingPlan, scale: float):
    lib = _lib.load()
    H, N, Dp = q.shape
    B = plan.block_size
    if B > MAX_BLOCK:
        raise ConfigError(f"block_size={B} > {MAX_BLOCK} is not supported by the compiled kernels")
    ensure_row_pos(plan)
    G = kv_group_of(q, k)
    out = torch.empty_like(q)
    lse = torch.empty((H, N), dtype=torch.float32, device=q.device)
    ws = _ws(lib.moba_fwd_workspace_size(H, N, Dp, B, plan.width), q.device)
    st = lib.moba_fwd_gqa(q.data_ptr(), k.data_ptr(), v.data_ptr(), H, G, N, Dp, B, plan.width,
                      plan.counts_d.data_ptr(), plan.offsets_d.data_ptr(), plan.flat_d.data_ptr(),
                      plan.row_pos.data_ptr(), float(scale), out.data_ptr(), lse.data_ptr(),
                      ws.data_ptr(), ws.numel(), _stream(q))
    _lib.check(st, "moba_fwd_gqa")
    return out, lse


def bwd(q, k, v, out, dout, lse, plan: RoutingPlan, scale: float, deterministic: bool = True):
    lib = _lib.load()
    H, N, Dp = q.shape
    B = plan.block_size
    if deterministic:
        ensure_row_pos(plan)
    G = kv_group_of(q, k)
    dq = torch.empty_like(q)
    dk = torch.empty_like(k)
    dv = torch.empty_like(v)
    ws = _ws(lib.moba_bwd_gqa_workspace_size(H, G, N, Dp, B, plan.width, int(deterministic)), q.device)
    st = lib.moba_bwd_gqa(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), dout.data_ptr(),
                      lse.data_ptr(), H, G, N, Dp, B, plan.width, plan.counts_d.data_ptr(),
                      plan.offsets_d.data_ptr(), plan.flat_d.data_ptr(),
                      _lib.ptr(plan.row_pos) if deterministic else None, int(deterministic), float(scale),
                      dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ws.data_ptr(), ws.numel(), _stream(q))
    _lib.check(st, "moba_bwd_gqa")
    return dq, dk, dv


def conv_bwd(k, conv_w, dk_conv):
    lib = _lib.load()
    H, N, Dp = k.shape
    width = int(conv_w.shape[0])
    conv_w = conv_w.to(device=k.device, dtype=torch.float32).contiguous()
    dk = torch.empty_like(k)
    dw = torch.empty((width, Dp), dtype=torch.float32, device=k.device)
    ws = _ws(lib.moba_conv_bwd_workspace_size(H, N, Dp, width), k.device)
    st = lib.moba_conv_bwd(k.data_ptr(), conv_w.data_ptr(), width, dk_conv.data_ptr(), H, N, Dp,
                           dk.data_ptr(), dw.data_ptr(), ws.data_ptr(), ws.numel(), _stream(k))
    _lib.check(st, "moba_conv_bwd")
    return dk, dw


def visible_pairs(plan: RoutingPlan) -> int:
    """Visible (query, key) pairs of a plan, computed on device: own block
    contributes i - jB + 1 keys, any other block its length."""
    t = plan.topk.long()
    N, B = plan.n_tokens, plan.block_size
    i = torch.arange(N, device=t.device).view(1, N, 1)
    own = i // B
    blen = torch.clamp(N - t * B, max=B)
    vis = torch.where(t == own, i - t * B + 1, blen)
    return int(torch.where(t >= 0, vis, torch.zeros_like(vis)).sum())


def scored_candidates(n_tokens: int, block_size: int) -> int:
    i = torch.arange(n_tokens, dtype=torch.int64)
    return int((i // block_size).sum())


def softmax_scale(d: int) -> float:
    return 1.0 / math.sqrt(d)
