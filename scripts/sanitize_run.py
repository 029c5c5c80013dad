"""One small invocation of every kernel on the hot path, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): centroids (+ key conv),
both routers (fp32 FFMA and tcgen05), varlen, the forward (d = 64 and 128,
B = 64 / 128 / 256), combine, both backward schedules and the conv backward.

usage: compute-sanitizer --tool racecheck python scripts/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2511_11571_b200 as mb  # noqa: E402
from paper_2511_11571_b200 import _device, _lib  # noqa: E402


def case(H, N, d, B, k, conv=0, route_mode=_lib.MOBA_ROUTE_TC, deterministic=False):
    g = torch.Generator(device="cuda").manual_seed(N + d + B + k)
    q, kk, v, do = (torch.randn(H, N, d, generator=g, device="cuda").bfloat16() for _ in range(4))
    w = (0.3 * torch.randn(conv, d, generator=g, device="cuda")).float() if conv else None
    cent, kc = _device.centroids(kk, B, w)
    plan = _device.route(q, cent, B, k, mode=route_mode)
    scale = _device.softmax_scale(d)
    out, lse = _device.fwd(q, kc, v, plan, scale)
    dq, dk, dv = _device.bwd(q, kc, v, out, do, lse, plan, scale,
                             deterministic=deterministic)
    if w is not None:
        _device.conv_bwd(kk, w, dk)
    torch.cuda.synchronize()
    print(f"case H={H} N={N} d={d} B={B} k={k} conv={conv} route={route_mode} det={deterministic}: "
          f"O {float(out.float().abs().mean()):.4f} dQ {float(dq.float().abs().mean()):.4f}", flush=True)


if __name__ == "__main__":
    torch.cuda.set_device(0)
    _lib.load()
    case(1, 640, 64, 128, 3)
    case(1, 640, 64, 128, 3, route_mode=_lib.MOBA_ROUTE_FP32, deterministic=True)
    case(1, 512, 128, 128, 2)
    case(1, 512, 64, 64, 4, conv=3)
    case(1, 700, 64, 256, 1)
    print("sanitize_run done")
