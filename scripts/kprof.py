"""Per-kernel device time of one eager MoBA fwd+bwd step (torch.profiler /
CUPTI), plus the tc router's recheck-queue length.

usage: python scripts/kprof.py H N d B k [mode] [reps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11571_b200 as mb  # noqa: E402
from paper_2511_11571_b200 import _device, _lib  # noqa: E402

H, N, d, B, k = (int(x) for x in sys.argv[1:6])
mode = sys.argv[6] if len(sys.argv) > 6 else "tc"
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 2
gen = torch.Generator(device="cuda").manual_seed(1234)
q, kk, v, do = (torch.randn(H, N, d, generator=gen, device="cuda").bfloat16() for _ in range(4))
for t in (q, kk, v):
    t.requires_grad_(True)


def step():
    for t in (q, kk, v):
        t.grad = None
    o = mb.moba_attn(q, kk, v, B, k, mode=mode)
    o.backward(do)


# recheck queue length of the tc router (last int region of the route workspace)
lib = _lib.load()
if mode == "tc":
    cent, _ = _device.centroids(kk.detach(), B)
    ws_bytes = lib.moba_route_workspace_size(H, N, B, k)
    ws = torch.zeros(ws_bytes, dtype=torch.uint8, device="cuda")
    n = -(-N // B)
    plan = _device._empty_plan(H, N, k + 1, n, q.device)
    st = lib.moba_route_gqa(q.detach().data_ptr(), cent.data_ptr(), H, 1, N, d, B, k, _lib.MOBA_ROUTE_TC,
                            *(t.data_ptr() for t in plan), ws.data_ptr(), ws_bytes,
                            torch.cuda.current_stream().cuda_stream)
    _lib.check(st, "route")
    torch.cuda.synchronize()
    rc_bytes = -(-((1 + H * N) * 4) // 256) * 256
    cnt = int(ws[ws_bytes - rc_bytes:ws_bytes - rc_bytes + 4].view(torch.int32).item())
    print(f"recheck rows: {cnt} of {H * N}")

for _ in range(2):
    step()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        step()
    torch.cuda.synchronize()
agg = {}
for e in prof.events():
    if e.device_type.name == "CUDA" and e.device_time > 0:
        a = agg.setdefault(e.name[:70], [0, 0.0])
        a[0] += 1
        a[1] += e.device_time
tot = sum(v[1] for v in agg.values()) / reps
print(f"H={H} N={N} d={d} B={B} k={k} mode={mode}: {tot / 1e3:.3f} ms of kernels per step")
for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {t / reps / 1e3:8.3f} ms  x{c / reps:4.1f}  {name}")
