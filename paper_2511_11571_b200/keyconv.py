"""Causal key short-conv with SiLU and residual, on the GPU (src/keyconv.py).

    k'[t] = k[t] + silu(sum_l W[l] * k[t - l])     (zero left pad)

The forward is the same kernel as the centroid stage (moba_centroids with a
conv weight), so in the attention path K' and the routing centroids come
out of one HBM pass. The backward is moba_conv_bwd.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device
from ._convert import from_heads, routing_heads, to_heads, to_weights
from .core import ShapeError


@dataclass
class ConvKernel:
    """Per-lag, per-channel weights, shape (width, d) (src/keyconv.py:22-40)."""

    weights: object

    def __post_init__(self):
        w = self.weights
        arr = w.detach().cpu().numpy() if isinstance(w, torch.Tensor) else np.asarray(w)
        if arr.ndim != 2:
            raise ShapeError("kernel weights must be 2-D (width x d)")
        if arr.shape[0] < 1:
            raise ShapeError("kernel width must be >= 1")
        if not np.all(np.isfinite(arr)):
            raise ShapeError("kernel weights must be finite")
        if arr.shape[0] > 5:
            raise ShapeError("kernel width > 5 is not supported by the compiled kernels")

    @property
    def width(self) -> int:
        return int(self.weights.shape[0])


def random_kernel(width: int, d: int, seed: int, dtype=np.float64) -> ConvKernel:
    """Fan-in init U(-1/sqrt(width), 1/sqrt(width)), seeded (src/keyconv.py:43-47)."""
    rng = np.random.default_rng(seed)
    bound = 1.0 / np.sqrt(width)
    return ConvKernel(rng.uniform(-bound, bound, size=(width, d)).astype(dtype))


def key_conv_forward(K, kernel: ConvKernel):
    """Transformed keys k + silu(conv(k)) (src/keyconv.py:70-78)."""
    if isinstance(K, np.ndarray) and K.ndim != 2:
        raise ShapeError("K must be 2-D (N x d)")
    k, info = to_heads(K, "K")
    k32 = routing_heads(K, "K", device=k.device)       # conv of the unrounded keys; K' is rounded once
    w = to_weights(kernel.weights, info.d, info.dp, k.device)
    # the conv is fused with the centroid pass (moba_centroids); a block of
    # 256 keys keeps that side output small
    _, k_conv = _device.centroids(k if k32 is None else k32, min(256, info.n_tokens), w)
    return from_heads(k_conv, info)


def key_conv_backward(K, kernel: ConvKernel, dK_out):
    """(dK, dW) of key_conv_forward (src/keyconv.py:81-104). dW is summed over
    heads when K carries several (one W shared across heads, src/cli.py:255-258)."""
    k, info = to_heads(K, "K")
    g, ginfo = to_heads(dK_out, "dK_out", device=k.device)
    if (ginfo.n_tokens, ginfo.d) != (info.n_tokens, info.d) or g.shape != k.shape:
        raise ShapeError(f"gradient shape does not match K")
    w = to_weights(kernel.weights, info.d, info.dp, k.device)
    dk, dw = _device.conv_bwd(k, w, g)
    dw = dw[:, : info.d]
    if info.kind == "numpy":
        dw = dw.cpu().numpy().astype(info.np_dtype)
    return from_heads(dk, info), dw
