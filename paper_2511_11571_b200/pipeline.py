"""Host-buffer MoBA fwd+bwd with the PCIe copies overlapped with the kernels.

`moba_fwd_bwd_host(q, k, v, do, block_size, top_k)` is the training-step
form of the drop-in for callers whose tensors live in (pinned) host memory,
e.g. the reference's own numpy callers (src/cli.py:276-280 loops heads on
the host; src/verification.py:165-166 runs fwd then bwd). It returns host
O, LSE, dQ, dK, dV — the same values as `moba_attn` + `.backward(do)`.

Heads are independent, so the heads are cut into chunks and
run as a three-stage pipeline on three CUDA streams:

  h2d stream      chunk c:   Q, K, V, dO  host -> HBM
  compute stream  chunk c:   centroids, route, varlen, fwd, combine, bwd
  d2h stream      chunk c:   O, LSE, dQ, dK, dV  HBM -> host

so chunk c+1's upload and chunk c-1's download overlap chunk c's kernels
(copy engines are independent of the SMs and the two PCIe directions are
full duplex). No value depends on the chunking: every kernel works per head.
"""

from __future__ import annotations

import torch

from . import _device
from .core import ConfigError, MobaConfig, ShapeError
from .router import ROUTE_MODES


def _chunks(H: int, n_chunks: int):
    n_chunks = max(1, min(int(n_chunks), H))
    base, rem = divmod(H, n_chunks)
    h0 = 0
    for c in range(n_chunks):
        h1 = h0 + base + (1 if c < rem else 0)
        yield h0, h1
        h0 = h1


class _GraphSlot:
    """A captured chunk step plus the events that guard its static buffers."""

    def __init__(self, step):
        self.step = step
        self.computed = None     # replay finished: inputs consumed, outputs written
        self.downloaded = None   # outputs copied to the host


class HostPipeline:
    """Reusable streams/events (and captured chunk graphs) for
    `moba_fwd_bwd_host` on one device."""

    def __init__(self, device=None):
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else
                                   torch.device(device).index or 0)
        self.h2d = torch.cuda.Stream(self.device)
        self.comp = torch.cuda.Stream(self.device)
        self.d2h = torch.cuda.Stream(self.device)
        self._slots: dict = {}

    def _graph_slots(self, key):
        """Two captured steps per chunk shape (double-buffered static inputs /
        outputs, so chunk c+1's upload and chunk c-1's download overlap chunk
        c's replay)."""
        slots = self._slots.get(key)
        if slots is None:
            from .graphs import MobaGraphedStep
            (hc, N, d), B, k, mode, det = key
            with torch.cuda.device(self.device):
                slots = [_GraphSlot(MobaGraphedStep((hc, N, d), B, k, mode=mode, deterministic=det,
                                                    device=self.device)) for _ in range(2)]
            self._slots[key] = slots
        return slots

    def run_graphed(self, q, k, v, do, block_size, top_k, *, n_chunks=4, mode="tc", deterministic=False,
                    out=None):
        """As `run`, but each chunk's kernels are one CUDA-graph replay (host
        cost per chunk: a few copies and one graph launch), which lets the
        heads be cut finer so the PCIe copies overlap more of the compute."""
        for name, t in (("q", q), ("k", k), ("v", v), ("do", do)):
            if t.is_cuda:
                raise ShapeError(f"{name} must be a host tensor for the host pipeline")
            if t.dim() != 3 or tuple(t.shape) != tuple(q.shape):
                raise ShapeError(f"{name} must be [H, N, d] like q, got {tuple(t.shape)}")
        H, N, d = q.shape
        MobaConfig(block_size_B=block_size, top_k=top_k, head_dim_d=d)
        if d not in _device.SUPPORTED_DP:
            raise ConfigError(f"host pipeline takes d in {_device.SUPPORTED_DP} (kernel layout), got {d}")
        if out is None:
            pin = torch.cuda.is_available()
            out = (torch.empty((H, N, d), dtype=torch.bfloat16, pin_memory=pin),
                   torch.empty((H, N), dtype=torch.float32, pin_memory=pin),
                   *(torch.empty((H, N, d), dtype=torch.bfloat16, pin_memory=pin) for _ in range(3)))
        o_h, lse_h, dq_h, dk_h, dv_h = out
        cur = torch.cuda.current_stream(self.device)
        for s in (self.h2d, self.comp, self.d2h):
            s.wait_stream(cur)
        uses = {}
        for h0, h1 in _chunks(H, n_chunks):
            key = ((h1 - h0, N, d), block_size, top_k, mode, deterministic)
            slots = self._graph_slots(key)
            u = uses.get(key, 0)
            uses[key] = u + 1
            sl = slots[u % 2]
            g = sl.step
            with torch.cuda.stream(self.h2d):
                if sl.computed is not None:
                    self.h2d.wait_event(sl.computed)
                for dst, src in ((g.q, q), (g.k, k), (g.v, v), (g.dout, do)):
                    with torch.no_grad():
                        dst.copy_(src[h0:h1], non_blocking=True)
                up = torch.cuda.Event()
                up.record(self.h2d)
            with torch.cuda.stream(self.comp):
                self.comp.wait_event(up)
                if sl.downloaded is not None:
                    self.comp.wait_event(sl.downloaded)
                g.replay()
                sl.computed = torch.cuda.Event()
                sl.computed.record(self.comp)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(sl.computed)
                dq, dk, dv = g.grads
                for src, dst in ((g.out, o_h), (g.lse, lse_h), (dq, dq_h), (dk, dk_h), (dv, dv_h)):
                    dst[h0:h1].copy_(src, non_blocking=True)
                sl.downloaded = torch.cuda.Event()
                sl.downloaded.record(self.d2h)
        cur.wait_stream(self.d2h)
        cur.wait_stream(self.comp)
        return o_h, lse_h, dq_h, dk_h, dv_h

    def run(self, q, k, v, do, block_size, top_k, *, n_chunks=4, mode="tc", deterministic=False, out=None):
        """q, k, v, do: host bf16 tensors [H, N, d] (pinned for real overlap).
        Returns host (o, lse, dq, dk, dv); `out` may pass preallocated pinned
        host buffers in that order. The copies are asynchronous: the call
        returns once they are enqueued and the current stream has been made to
        wait for them, so the host buffers hold the results after
        `torch.cuda.current_stream().synchronize()` (moba_fwd_bwd_host does
        that unless synchronize=False)."""
        for name, t in (("q", q), ("k", k), ("v", v), ("do", do)):
            if t.is_cuda:
                raise ShapeError(f"{name} must be a host tensor for the host pipeline")
            if t.dim() != 3 or tuple(t.shape) != tuple(q.shape):
                raise ShapeError(f"{name} must be [H, N, d] like q, got {tuple(t.shape)}")
        H, N, d = q.shape
        MobaConfig(block_size_B=block_size, top_k=top_k, head_dim_d=d)
        if d not in _device.SUPPORTED_DP:
            raise ConfigError(f"host pipeline takes d in {_device.SUPPORTED_DP} (kernel layout), got {d}")
        if out is None:
            pin = torch.cuda.is_available()
            out = (torch.empty((H, N, d), dtype=torch.bfloat16, pin_memory=pin),
                   torch.empty((H, N), dtype=torch.float32, pin_memory=pin),
                   *(torch.empty((H, N, d), dtype=torch.bfloat16, pin_memory=pin) for _ in range(3)))
        o_h, lse_h, dq_h, dk_h, dv_h = out
        scale = _device.softmax_scale(d)
        route_mode = ROUTE_MODES[mode]
        cur = torch.cuda.current_stream(self.device)
        for s in (self.h2d, self.comp, self.d2h):
            s.wait_stream(cur)
        keep = []
        for h0, h1 in _chunks(H, n_chunks):
            with torch.cuda.stream(self.h2d):
                xs = [t[h0:h1].to(self.device, non_blocking=True) for t in (q, k, v, do)]
                up = torch.cuda.Event()
                up.record(self.h2d)
            with torch.cuda.stream(self.comp):
                self.comp.wait_event(up)
                for x in xs:
                    x.record_stream(self.comp)
                qd, kd, vd, dod = xs
                cent, _ = _device.centroids(kd, block_size)
                plan = _device.route(qd, cent, block_size, top_k, route_mode)
                o, lse = _device.fwd(qd, kd, vd, plan, scale)
                dq, dk, dv = _device.bwd(qd, kd, vd, o, dod, lse, plan, scale, deterministic=deterministic)
                done = torch.cuda.Event()
                done.record(self.comp)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(done)
                for src, dst in ((o, o_h), (lse, lse_h), (dq, dq_h), (dk, dk_h), (dv, dv_h)):
                    src.record_stream(self.d2h)
                    dst[h0:h1].copy_(src, non_blocking=True)
            keep.append((xs, o, lse, dq, dk, dv))
        cur.wait_stream(self.d2h)
        cur.wait_stream(self.comp)
        return o_h, lse_h, dq_h, dk_h, dv_h


_PIPELINES: dict = {}


def moba_fwd_bwd_host(q, k, v, do, block_size: int, top_k: int, *, n_chunks: int | None = None, mode: str = "tc",
                      deterministic: bool = False, out=None, synchronize: bool = True, graphs: bool = True):
    """MoBA forward + backward on host tensors with overlapped PCIe copies.

    q, k, v, do: bf16 host tensors [H, N, d], d in {64, 128}. Returns host
    (O, LSE, dQ, dK, dV). Requires a CUDA device (no CPU fallback).
    graphs=True replays one captured CUDA graph per head chunk (captured on
    first use for each chunk shape), graphs=False launches the kernels
    eagerly. Default chunking: about 32 MB of inputs per chunk, at least 4
    chunks (measured on PCIe 5, graphs: 16 x 8K heads 1.99 / 2.05 / 2.73 ms
    at 4 / 8 / 16 chunks; 32 x 64K heads 25.9 / 26.0 / 24.3 ms at 8 / 16 / 32
    chunks — the last chunk's download is the exposed tail)."""
    if n_chunks is None:
        in_bytes = sum(t.numel() * t.element_size() for t in (q, k, v, do))
        n_chunks = max(4, int(round(in_bytes / (32 << 20)))) if graphs else 4
        n_chunks = min(n_chunks, int(q.shape[0]))
    if not torch.cuda.is_available():
        raise ConfigError("moba_fwd_bwd_host needs a CUDA device (there is no CPU fallback)")
    dev = torch.cuda.current_device()
    pipe = _PIPELINES.get(dev)
    if pipe is None:
        pipe = _PIPELINES[dev] = HostPipeline(dev)
    runner = pipe.run_graphed if graphs else pipe.run
    res = runner(q, k, v, do, block_size, top_k, n_chunks=n_chunks, mode=mode, deterministic=deterministic, out=out)
    if synchronize:
        torch.cuda.current_stream(dev).synchronize()
    return res
