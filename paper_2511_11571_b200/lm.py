"""The paper's hybrid MoBA language model (SURVEY.md §8 f2, configs[4]).

PAPER.md:313-314: 24 layers; odd layers (1st, 3rd, ...) use sliding-window
attention (window 256) with RoPE, even layers use MoBA without positional
encoding (optionally with the causal key short-conv, kconv3 / kconv5);
340M family = hidden 1024, 16 heads, head dim 64, SwiGLU MLP with
intermediate size 2816, 32K vocabulary.

This module is the caller of the hot path, not part of it: the MoBA layers
call `moba_attn` (the sm_100a kernels of this package, autograd through
`MobaAttnFunction`); the sliding-window layers call FlashAttention-2's
windowed kernel (library code, the same role FA plays in the reference
setup); norms, projections, MLP and the loss are plain PyTorch. Weights are
randomly initialised and tokens synthetic (no checkpoints / datasets here).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.nn as nn
import torch.nn.functional as F

from .attention import moba_attn


@dataclass
class MobaLMConfig:
    vocab: int = 32000
    hidden: int = 1024
    heads: int = 16
    head_dim: int = 64
    intermediate: int = 2816
    layers: int = 24
    swa_window: int = 256
    block_size: int = 128
    top_k: int = 8
    conv_width: int = 0          # 0, 3 (kconv3) or 5 (kconv5) on the MoBA layers
    rope_base: float = 10000.0
    route_mode: str = "tc"
    swa_impl: str = "flash"      # "flash" (FA2 windowed kernel) or "torch" (masked SDPA; tests, fp32 models)


def _rope(x: torch.Tensor, base: float) -> torch.Tensor:
    """Rotary embedding on [b, N, h, d] (rotate-half convention)."""
    b, N, h, d = x.shape
    half = d // 2
    inv = 1.0 / (base ** (torch.arange(0, half, device=x.device, dtype=torch.float32) / half))
    ang = torch.arange(N, device=x.device, dtype=torch.float32)[:, None] * inv[None, :]
    cos, sin = ang.cos()[None, :, None, :], ang.sin()[None, :, None, :]
    x1, x2 = x[..., :half].float(), x[..., half:].float()
    return torch.cat((x1 * cos - x2 * sin, x1 * sin + x2 * cos), dim=-1).to(x.dtype)


class Attention(nn.Module):
    def __init__(self, cfg: MobaLMConfig, moba: bool):
        super().__init__()
        self.cfg, self.moba = cfg, moba
        self.moba_fn = moba_attn     # the MoBA operator (a test may swap in a reference implementation)
        inner = cfg.heads * cfg.head_dim
        self.qkv = nn.Linear(cfg.hidden, 3 * inner, bias=False)
        self.out = nn.Linear(inner, cfg.hidden, bias=False)
        self.conv = None
        if moba and cfg.conv_width:
            bound = 1.0 / math.sqrt(cfg.conv_width)      # src/keyconv.py:43-47
            self.conv = nn.Parameter(torch.empty(cfg.conv_width, cfg.head_dim).uniform_(-bound, bound))

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        b, N, _ = x.shape
        c = self.cfg
        q, k, v = self.qkv(x).view(b, N, 3, c.heads, c.head_dim).unbind(2)
        if self.moba:
            # MoBA layer: no positional encoding; [b, h, N, d] for the kernels
            # (bf16 operands; the output returns to the model's dtype)
            o = self.moba_fn(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2), c.block_size, c.top_k,
                             conv_weight=self.conv, mode=c.route_mode)
            o = o.transpose(1, 2).to(x.dtype)
        elif c.swa_impl == "flash":
            from flash_attn import flash_attn_func
            q, k = _rope(q, c.rope_base), _rope(k, c.rope_base)
            o = flash_attn_func(q, k, v, causal=True, window_size=(c.swa_window - 1, 0))
        else:
            q, k = _rope(q, c.rope_base), _rope(k, c.rope_base)
            i = torch.arange(N, device=x.device)
            keep = (i[None, :] <= i[:, None]) & (i[:, None] - i[None, :] < c.swa_window)
            o = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2),
                                               attn_mask=keep).transpose(1, 2)
        return self.out(o.reshape(b, N, c.heads * c.head_dim))


class MLP(nn.Module):
    def __init__(self, cfg: MobaLMConfig):
        super().__init__()
        self.gate_up = nn.Linear(cfg.hidden, 2 * cfg.intermediate, bias=False)
        self.down = nn.Linear(cfg.intermediate, cfg.hidden, bias=False)

    def forward(self, x):
        g, u = self.gate_up(x).chunk(2, dim=-1)
        return self.down(F.silu(g) * u)


class Block(nn.Module):
    def __init__(self, cfg: MobaLMConfig, moba: bool):
        super().__init__()
        self.n1 = nn.RMSNorm(cfg.hidden)
        self.attn = Attention(cfg, moba)
        self.n2 = nn.RMSNorm(cfg.hidden)
        self.mlp = MLP(cfg)

    def forward(self, x):
        x = x + self.attn(self.n1(x))
        return x + self.mlp(self.n2(x))


class MobaLM(nn.Module):
    """Layer i (1-based) is sliding-window if i is odd, MoBA if i is even."""

    def __init__(self, cfg: MobaLMConfig):
        super().__init__()
        self.cfg = cfg
        self.embed = nn.Embedding(cfg.vocab, cfg.hidden)
        self.blocks = nn.ModuleList(Block(cfg, moba=(i % 2 == 0)) for i in range(1, cfg.layers + 1))
        self.norm = nn.RMSNorm(cfg.hidden)
        self.head = nn.Linear(cfg.hidden, cfg.vocab, bias=False)
        for m in self.modules():
            if isinstance(m, nn.Linear):
                nn.init.normal_(m.weight, std=0.02)
            elif isinstance(m, nn.Embedding):
                nn.init.normal_(m.weight, std=0.02)

    def n_params(self) -> int:
        return sum(p.numel() for p in self.parameters())

    def forward(self, tokens: torch.Tensor) -> torch.Tensor:
        x = self.embed(tokens)
        for blk in self.blocks:
            x = blk(x)
        return self.head(self.norm(x))

    def loss(self, tokens: torch.Tensor, loss_chunk: int = 8192) -> torch.Tensor:
        """Next-token cross-entropy; the vocabulary projection and the loss run
        in sequence chunks so the [N, vocab] logits never exist at once."""
        x = self.embed(tokens)
        for blk in self.blocks:
            x = blk(x)
        h = self.norm(x)[:, :-1]
        tgt = tokens[:, 1:]
        total = h.new_zeros((), dtype=torch.float32)
        n = tgt.numel()
        for s in range(0, h.shape[1], loss_chunk):
            logits = self.head(h[:, s:s + loss_chunk]).float()
            total = total + F.cross_entropy(logits.reshape(-1, logits.shape[-1]),
                                            tgt[:, s:s + loss_chunk].reshape(-1), reduction="sum")
        return total / n


def train_step(model: MobaLM, opt: torch.optim.Optimizer, tokens: torch.Tensor) -> torch.Tensor:
    """One optimizer step (forward, loss, backward, AdamW update). Returns the
    loss (a device tensor; no host sync)."""
    opt.zero_grad(set_to_none=True)
    loss = model.loss(tokens)
    loss.backward()
    opt.step()
    return loss.detach()


def model_flops_per_token(cfg: MobaLMConfig, seq: int) -> float:
    """Training FLOPs per token (fwd + bwd = 3x fwd): 6 x dense parameters
    (projections, MLP, LM head) plus the attention matmuls — MoBA layers
    14*d*P/N per token per head (P visible pairs, fwd+bwd) and SWA layers the
    same with a window of w keys."""
    h, d, H, I, V = cfg.hidden, cfg.head_dim, cfg.heads, cfg.intermediate, cfg.vocab
    per_layer = 2 * h * 3 * H * d + 2 * H * d * h + 2 * h * 2 * I + 2 * I * h
    dense = 3 * (cfg.layers * per_layer + 2 * h * V)
    B, k = cfg.block_size, cfg.top_k
    vis_moba = sum(min(k, i // B) * B + (i % B) + 1 for i in range(seq)) / seq
    vis_swa = sum(min(i + 1, cfg.swa_window) for i in range(seq)) / seq
    n_moba = cfg.layers // 2
    attn = 14 * d * H * (n_moba * vis_moba + (cfg.layers - n_moba) * vis_swa)
    return dense + attn
