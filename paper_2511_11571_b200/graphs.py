"""CUDA-graph replay of a MoBA attention training step.

A step is `moba_attn(q, k, v, B, top_k)` followed by `out.backward(dout)` —
centroids, routing, varlen plan, forward, combine, backward, dQ finalize:
~15 dependent kernels. Launched eagerly, each carries a few microseconds of
launch latency between kernels; captured once into a CUDA graph and replayed,
the whole step is submitted as one unit (the same kernels, the same work,
the same results).

`MobaGraphedStep(shape, block_size, top_k)` owns static input buffers;
`step(q, k, v, dout)` copies new inputs in (device-to-device) and replays.
Shapes, block size, top-k and mode are fixed per instance (a graph bakes its
launch geometry), which is the situation of a training loop.
"""

from __future__ import annotations

import torch

from . import _lib
from .attention import moba_attn
from .core import ConfigError


class MobaGraphedStep:
    """Captured fwd+bwd of `moba_attn` for fixed [..., N, d] bf16 shapes."""

    def __init__(self, shape, block_size: int, top_k: int, *, mode: str = "tc", deterministic: bool = False,
                 conv_weight: torch.Tensor | None = None, device=None, warmup: int = 2):
        if not torch.cuda.is_available():
            raise ConfigError("MobaGraphedStep needs a CUDA device (there is no CPU fallback)")
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.block_size, self.top_k, self.mode, self.deterministic = block_size, top_k, mode, deterministic
        # warm-up / capture inputs: seeded random values (all-zero inputs make
        # every routing score tie, which sends every row to the exact fp32
        # re-routing pass — correct, but a needlessly slow warm-up)
        gen = torch.Generator(device=dev).manual_seed(0)
        mk = lambda: torch.randn(tuple(shape), generator=gen, device=dev).to(torch.bfloat16)
        self.q, self.k, self.v, self.dout = mk().requires_grad_(True), mk().requires_grad_(True), \
            mk().requires_grad_(True), mk()
        self.conv_weight = None if conv_weight is None else conv_weight.detach().clone().requires_grad_(True)
        lib = _lib.load()
        timing = lib.moba_timing_enabled()
        lib.moba_timing_enable(0)   # per-stage CUDA-event timers are not captured
        try:
            self._capture(dev, lib, warmup)
        finally:
            lib.moba_timing_enable(timing)

    def _capture(self, dev, lib, warmup):
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for _ in range(max(1, warmup)):
                self._body()
        torch.cuda.current_stream(dev).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        n0 = lib.moba_launch_count()
        self._zero_grads()
        with torch.cuda.graph(self.graph):
            self.out, self.lse = self._body()
        self.launches_per_step = int(lib.moba_launch_count() - n0)

    def _zero_grads(self):
        for t in (self.q, self.k, self.v, self.conv_weight):
            if t is not None:
                t.grad = None

    def _body(self):
        self._zero_grads()
        out, lse = moba_attn(self.q, self.k, self.v, self.block_size, self.top_k, conv_weight=self.conv_weight,
                             mode=self.mode, deterministic=self.deterministic, return_lse=True)
        out.backward(self.dout)
        return out, lse

    def replay(self):
        """Re-run the captured step on the current contents of the static
        buffers (on the current stream)."""
        self.graph.replay()

    @property
    def grads(self):
        return self.q.grad, self.k.grad, self.v.grad

    def step(self, q=None, k=None, v=None, dout=None):
        """Copy new inputs (device tensors of the captured shape) and replay.
        Returns (out, dq, dk, dv) — views of the graph's static outputs, valid
        until the next replay."""
        with torch.no_grad():
            for dst, src in ((self.q, q), (self.k, k), (self.v, v), (self.dout, dout)):
                if src is not None:
                    dst.copy_(src, non_blocking=True)
        self.graph.replay()
        return self.out, self.q.grad, self.k.grad, self.v.grad
