"""MoBA attention on the GPU — the drop-in for src/attention.py.

Reference-shaped entry points (same names, argument meaning, errors):
  moba_attention(Q, K, V, cfg, counters=None, threads=1)  (src/attention.py:305-314)
  moba_forward(Q, K, V, plan, cfg, counters=None, threads=1)  (src/attention.py:147-182)
  moba_backward(Q, K, V, O, dO, lse, plan, cfg, counters=None,
                schedule="deterministic")  (src/attention.py:239-302)
plus the torch-facing, autograd-enabled batched call used by training code:
  moba_attn(q, k, v, block_size, top_k, causal=True, conv_weight=None)

Numerics: the attention kernels compute in bf16 with fp32 accumulation and
fp32 LSE; f32/f64 inputs are rounded to bf16 for the attention operands
(the tolerance contract is max-abs 2e-2 / rel-L2 1e-2 against the reference
on the same inputs), while centroids and fp32-mode routing use the unrounded
values, so block selection matches the reference up to score ties.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device
from ._convert import from_heads, routing_heads, to_heads, to_weights
from .core import (ConfigError, MobaConfig, OpCounters, PlanValidationError, RoutingPlan, ShapeError,
                   resolve_threads)
from .counters import add_backward_counters, add_forward_counters, add_plan_counters
from .router import ROUTE_MODES, build_plan


@dataclass
class AttentionOutput:
    """Attention result: output rows plus per-query natural-log LSE over the
    scaled scores (src/reference.py:21-26)."""

    output: object
    logsumexp: object


def _check_qkv(Q, K, V):
    # src/reference.py:29-33
    for x in (Q, K, V):
        if isinstance(x, np.ndarray) and x.ndim != 2:
            raise ShapeError("Q, K, V must be 2-D (N x d)")
    if tuple(Q.shape) != tuple(K.shape) or tuple(K.shape) != tuple(V.shape):
        raise ShapeError(f"shape mismatch: Q{tuple(Q.shape)} K{tuple(K.shape)} V{tuple(V.shape)}")


_PLAN_FIELDS = ("topk_indices", "counts", "offsets", "flat_queries")


def _as_device_plan(plan, info, cfg: MobaConfig, device) -> RoutingPlan:
    """A plan built elsewhere — e.g. the reference's own RoutingPlan dataclass
    (src/core.py:229-251: topk_indices, counts, offsets, flat_queries as
    numpy arrays, one head) — uploaded as this package's device plan; its
    invariants are then checked by validate_plan like any other plan."""
    if not all(hasattr(plan, f) for f in _PLAN_FIELDS):
        raise PlanValidationError("plan must be a RoutingPlan (this package's, or one with the reference's "
                                  "topk_indices / counts / offsets / flat_queries fields)")
    try:
        arrs = [np.asarray(getattr(plan, f)) for f in _PLAN_FIELDS]
    except Exception as e:  # pragma: no cover - exotic array types
        raise PlanValidationError(f"plan fields are not arrays: {e}") from None
    topk, counts, offsets, flat = arrs
    if topk.ndim == 2:                      # the reference's per-head plan
        topk, counts, offsets, flat = topk[None], counts[None], offsets[None], flat[None]
    if topk.ndim != 3 or counts.ndim != 2 or offsets.ndim != 2 or flat.ndim != 2:
        raise PlanValidationError("plan arrays have unexpected ranks")
    H, N, width = topk.shape
    if N != info.n_tokens:
        raise PlanValidationError(f"topk_indices shape {tuple(topk.shape)} does not match N={info.n_tokens}")
    if counts.shape[0] != H or np.any(counts.astype(np.int64).sum(axis=1) != flat.shape[1]):
        raise PlanValidationError("flat_queries length does not match sum(counts)")
    if flat.shape[1] > N * width:
        raise PlanValidationError("non-sentinel entry count does not match sum(counts)")
    flat_cap = np.full((H, N * width), -1, dtype=np.int32)
    flat_cap[:, : flat.shape[1]] = flat[:, : N * width]
    up = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32), device=device)
    return RoutingPlan(up(topk), up(counts), up(offsets), up(flat_cap), None, N, cfg.block_size_B)


def _prepare_plan(plan, info, cfg: MobaConfig, H: int, device) -> RoutingPlan:
    if not isinstance(plan, RoutingPlan):
        plan = _as_device_plan(plan, info, cfg, device)
    if plan.n_heads != H:
        raise PlanValidationError(f"plan has {plan.n_heads} heads, inputs have {H}")
    _device.validate(plan, info.n_tokens, cfg.block_size_B)
    plan.block_size = cfg.block_size_B
    return plan


def moba_forward(Q, K, V, plan: RoutingPlan, cfg: MobaConfig,
                 counters: OpCounters | None = None, threads: int | None = 1) -> AttentionOutput:
    """Plan-driven attention forward (src/attention.py:147-182)."""
    _check_qkv(Q, K, V)
    resolve_threads(threads)
    q, info = to_heads(Q, "Q")
    k, _ = to_heads(K, "K", device=q.device)
    v, _ = to_heads(V, "V", device=q.device)
    plan = _prepare_plan(plan, info, cfg, q.shape[0], q.device)
    out, lse = _device.fwd(q, k, v, plan, _device.softmax_scale(info.d))
    if counters is not None:
        add_forward_counters(counters, plan, info.d, cfg, _device.visible_pairs(plan))
    return AttentionOutput(from_heads(out, info), from_heads(lse, info, channels=False))


def moba_backward(Q, K, V, O, dO, lse, plan: RoutingPlan, cfg: MobaConfig,
                  counters: OpCounters | None = None, schedule: str = "deterministic"):
    """Plan-driven backward with score recomputation (src/attention.py:239-302).

    schedule="deterministic" sums each query's per-block dQ partials in slot
    order (bitwise repeatable); "parallel" accumulates dQ with fp32 vector
    reductions (rounding may vary run to run), like the reference's parallel
    schedule (src/attention.py:276-293).
    """
    _check_qkv(Q, K, V)
    if tuple(O.shape) != tuple(Q.shape) or tuple(dO.shape) != tuple(Q.shape):
        raise ShapeError("O and dO must match Q's shape")
    q, info = to_heads(Q, "Q")
    N = info.n_tokens
    lse_t = lse if isinstance(lse, torch.Tensor) else torch.as_tensor(np.asarray(lse, dtype=np.float64))
    if tuple(lse_t.shape) != (*info.lead, N):
        raise PlanValidationError(f"logsumexp has shape {tuple(lse_t.shape)}, expected {(*info.lead, N)}")
    lse_t = lse_t.to(device=q.device, dtype=torch.float32).reshape(-1, N).contiguous()
    if not bool(torch.isfinite(lse_t).all()):
        raise PlanValidationError("logsumexp contains non-finite entries")
    if schedule not in ("deterministic", "parallel"):
        raise ValueError(f"unknown schedule {schedule!r}")
    k, _ = to_heads(K, "K", device=q.device)
    v, _ = to_heads(V, "V", device=q.device)
    o, _ = to_heads(O, "O", device=q.device)
    do, _ = to_heads(dO, "dO", device=q.device)
    plan = _prepare_plan(plan, info, cfg, q.shape[0], q.device)
    dq, dk, dv = _device.bwd(q, k, v, o, do, lse_t, plan, _device.softmax_scale(info.d),
                             deterministic=(schedule == "deterministic"))
    if counters is not None:
        add_backward_counters(counters, plan, info.d, cfg, _device.visible_pairs(plan))
    return from_heads(dq, info), from_heads(dk, info), from_heads(dv, info)


def moba_attention(Q, K, V, cfg: MobaConfig, counters: OpCounters | None = None,
                   threads: int | None = 1, mode: str = "fp32", kernel=None) -> tuple[AttentionOutput, RoutingPlan]:
    """End-to-end routed attention: centroids, tiled top-k, varlen, forward
    (src/attention.py:305-314). Routing uses the UNSCALED Q (src/attention.py:312).
    `kernel` (a ConvKernel, optional) applies the key short-conv first, fused
    with the centroids so routing sees the unrounded K' (what the reference's
    CLI does with key_conv_forward before moba_attention, src/cli.py:277-278)."""
    _check_qkv(Q, K, V)
    if Q.shape[-1] != cfg.head_dim_d:
        raise ShapeError(f"d={Q.shape[-1]} does not match cfg.head_dim_d={cfg.head_dim_d}")
    resolve_threads(threads)
    q, info = to_heads(Q, "Q")
    k, _ = to_heads(K, "K", device=q.device)
    v, _ = to_heads(V, "V", device=q.device)
    k32 = routing_heads(K, "K", device=q.device)       # unrounded keys for the centroids (non-bf16 callers)
    k_src = k if k32 is None else k32
    if kernel is not None:
        w = to_weights(getattr(kernel, "weights", kernel), info.d, info.dp, q.device)
        cent, k = _device.centroids(k_src, cfg.block_size_B, w)
    else:
        cent, _ = _device.centroids(k_src, cfg.block_size_B)
    if cfg.top_k > _device.MAX_TOP_K:
        raise ConfigError(f"top_k={cfg.top_k} is not supported by the compiled kernels")
    q32 = routing_heads(Q, "Q", device=q.device) if mode == "fp32" else None
    plan = _device.route(q if q32 is None else q32, cent, cfg.block_size_B, cfg.top_k, ROUTE_MODES[mode])
    out, lse = _device.fwd(q, k, v, plan, _device.softmax_scale(info.d))
    if counters is not None:    # build_plan + moba_forward (src/attention.py:312-313)
        add_plan_counters(counters, q.shape[0], info.n_tokens, info.d, cfg.block_size_B, cfg.phys_tile_Br)
        add_forward_counters(counters, plan, info.d, cfg, _device.visible_pairs(plan))
    return AttentionOutput(from_heads(out, info), from_heads(lse, info, channels=False)), plan


# --------------------------------------------------------------------------
# autograd-enabled batched call
# --------------------------------------------------------------------------

class MobaAttnFunction(torch.autograd.Function):
    """q, k, v: bf16 CUDA [H, N, Dp] (kernel layout). The routing plan is
    built in forward and frozen for backward (src/verification.py:168-169);
    routing receives no gradient."""

    @staticmethod
    def forward(ctx, q, k, v, conv_w, block_size, top_k, scale, mode, deterministic):
        cent, k_used = _device.centroids(k, block_size, conv_w)
        plan = _device.route(q, cent, block_size, top_k, mode)
        out, lse = _device.fwd(q, k_used, v, plan, scale)
        ctx.save_for_backward(q, k, k_used, v, out, lse, conv_w if conv_w is not None else torch.empty(0))
        ctx.plan = plan
        ctx.scale = scale
        ctx.has_conv = conv_w is not None
        ctx.deterministic = deterministic
        ctx.mark_non_differentiable(lse)
        return out, lse

    @staticmethod
    def backward(ctx, dout, _dlse):
        q, k, k_used, v, out, lse, conv_w = ctx.saved_tensors
        dq, dk_used, dv = _device.bwd(q, k_used, v, out, dout.contiguous(), lse, ctx.plan, ctx.scale,
                                      deterministic=ctx.deterministic)
        dw = None
        if ctx.has_conv:
            dk, dw = _device.conv_bwd(k, conv_w, dk_used)
        else:
            dk = dk_used
        return dq, dk, dv, dw, None, None, None, None, None


def _check_gqa(q, k, v):
    """q [..., Hq, N, d]; k, v [..., Hkv, N, d] with Hq a multiple of Hkv
    (GQA; Hkv = 1 is MQA; Hkv = Hq is the reference's MHA)."""
    if tuple(k.shape) != tuple(v.shape):
        raise ShapeError(f"k{tuple(k.shape)} and v{tuple(v.shape)} must match")
    if q.dim() < 2 or k.dim() != q.dim():
        raise ShapeError(f"q{tuple(q.shape)} and k{tuple(k.shape)} must have the same rank (>= 2)")
    if tuple(k.shape) == tuple(q.shape):
        return
    if q.dim() < 3 or q.shape[:-3] != k.shape[:-3] or q.shape[-2:] != k.shape[-2:] or q.shape[-3] % k.shape[-3]:
        raise ShapeError(f"GQA needs q[..., Hq, N, d] and k/v[..., Hkv, N, d] with Hkv dividing Hq, "
                         f"got q{tuple(q.shape)} k{tuple(k.shape)}")


def moba_attn(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, block_size: int, top_k: int,
              causal: bool = True, conv_weight: torch.Tensor | None = None, mode: str = "fp32",
              deterministic: bool = False, return_lse: bool = False):
    """Batched MoBA attention for bf16 CUDA tensors [..., N, d] (d <= 128).
    k and v may have fewer heads than q (GQA/MQA, [..., Hkv, N, d]): query
    head h uses K/V head h // (Hq / Hkv) for routing and attention, and dK /
    dV are summed over the query heads sharing a K/V head.

    The north-star facade (q, k, v, block size B, top-k, causal). Only causal
    attention exists in the reference (src/attention.py:127-133), so
    causal=False raises ConfigError. conv_weight [width, d] applies the key
    short-conv before routing and attention (src/cli.py:277-278).
    """
    if not causal:
        raise ConfigError("MoBA attention is causal only (src/attention.py:127-133)")
    MobaConfig(block_size_B=block_size, top_k=top_k, head_dim_d=q.shape[-1],
               conv_width=0 if conv_weight is None else int(conv_weight.shape[0]))
    _check_gqa(q, k, v)
    for name, t in (("q", q), ("k", k), ("v", v)):
        _device.require_cuda(t, name)
    lead, N, d = tuple(q.shape[:-2]), q.shape[-2], q.shape[-1]
    dp = _device.padded_dim(d)

    def kern(t):
        t = t.to(torch.bfloat16).reshape(-1, N, d)
        return torch.nn.functional.pad(t, (0, dp - d)) if dp != d else t.contiguous()

    w = None
    if conv_weight is not None:
        w = conv_weight.to(device=q.device, dtype=torch.float32)
        if dp != d:
            w = torch.nn.functional.pad(w, (0, dp - d))
        w = w.contiguous()
    # GQA / MQA: k, v flatten to [batch * Hkv, N, d]; flat query head i maps
    # to flat K/V head i // (Hq / Hkv) (batch-major flattening keeps that exact)
    out, lse = MobaAttnFunction.apply(kern(q), kern(k), kern(v), w, block_size, top_k,
                                      _device.softmax_scale(d), ROUTE_MODES[mode], deterministic)
    out = out[..., :d].reshape(*lead, N, d)
    if return_lse:
        return out, lse.reshape(*lead, N)
    return out
