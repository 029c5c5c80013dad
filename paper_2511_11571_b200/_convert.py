"""Host <-> kernel-layout conversion.

The reference's operators take 2-D numpy arrays [N, d] per head
(src/reference.py:29-33). The drop-in accepts those (results come back as
numpy in the input's float dtype) and, for the fast path, torch tensors of
shape [N, d], [H, N, d] or [b, H, N, d] (results stay on the GPU in bf16 /
fp32). Internally the attention operands are bf16 [H, N, Dp] with Dp in
{64, 128}; the extra channels are zero, which leaves every dot product
unchanged. Callers whose Q / K are not bf16 (numpy f32 / f64, torch fp32 /
fp64 / fp16) also get an fp32 copy: centroids and routing are computed from
the unrounded values (to_heads_f32), so the block selection is not moved by
the bf16 rounding of the attention operands.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from ._device import padded_dim
from .core import ShapeError


@dataclass
class HeadsInfo:
    kind: str            # "numpy" or "torch"
    lead: tuple          # leading dims before [N, d]
    n_tokens: int
    d: int
    dp: int
    np_dtype: object = None
    device: object = None


def _device_for(x):
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return x.device
    return torch.device("cuda", torch.cuda.current_device())


def to_heads(x, name: str = "tensor", device=None, dtype=torch.bfloat16):
    """-> (CUDA tensor [H, N, Dp] of `dtype` (bf16 by default), HeadsInfo)."""
    if isinstance(x, np.ndarray) or not isinstance(x, torch.Tensor):
        arr = np.asarray(x)
        if arr.ndim < 2:
            raise ShapeError(f"{name} must be at least 2-D (N x d), got shape {arr.shape}")
        if not np.issubdtype(arr.dtype, np.floating):
            raise ShapeError(f"{name} must be floating point, got {arr.dtype}")
        info = HeadsInfo("numpy", arr.shape[:-2], arr.shape[-2], arr.shape[-1], padded_dim(arr.shape[-1]),
                         np_dtype=arr.dtype)
        dev = device or _device_for(None)
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).to(dev)
    else:
        if x.dim() < 2:
            raise ShapeError(f"{name} must be at least 2-D (N x d), got shape {tuple(x.shape)}")
        info = HeadsInfo("torch", tuple(x.shape[:-2]), x.shape[-2], x.shape[-1], padded_dim(x.shape[-1]))
        dev = device or _device_for(x)
        t = x.to(dev)
    info.device = dev
    t = t.to(dtype).reshape(-1, info.n_tokens, info.d)
    if info.dp != info.d:
        t = torch.nn.functional.pad(t, (0, info.dp - info.d))
    return t.contiguous(), info


def needs_fp32_routing(x) -> bool:
    """True unless x is already bf16 (then rounding it changes nothing)."""
    return not (isinstance(x, torch.Tensor) and x.dtype == torch.bfloat16)


def routing_heads(x, name: str, device=None):
    """fp32 [H, N, Dp] copy for centroids / routing when x is not bf16, else None."""
    if not needs_fp32_routing(x):
        return None
    t, _ = to_heads(x, name, device=device, dtype=torch.float32)
    return t


def from_heads(t: torch.Tensor, info: HeadsInfo, channels: bool = True):
    """Kernel layout -> caller layout ([..., N, d] or [..., N] for channels=False)."""
    if channels:
        t = t[..., : info.d].reshape(*info.lead, info.n_tokens, info.d)
    else:
        t = t.reshape(*info.lead, info.n_tokens)
    if info.kind == "numpy":
        return t.float().cpu().numpy().astype(info.np_dtype)
    return t


def to_weights(w, d: int, dp: int, device) -> torch.Tensor:
    """Conv weights [width, d] -> fp32 CUDA [width, Dp] (zero padded)."""
    if isinstance(w, torch.Tensor):
        t = w.detach().to(device=device, dtype=torch.float32)
    else:
        t = torch.as_tensor(np.asarray(w, dtype=np.float32), device=device)
    if t.dim() != 2 or t.shape[1] != d:
        raise ShapeError(f"kernel channels {tuple(t.shape)} do not match d={d}")
    if dp != d:
        t = torch.nn.functional.pad(t, (0, dp - d))
    return t.contiguous()
