import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11571_b200 import _device, _lib
lib = _lib.load()
for (H, N, d, B, k) in [(16, 8192, 64, 128, 8), (32, 65536, 64, 128, 8)]:
    torch.manual_seed(0)
    q, kk, v = (torch.randn(H, N, d, device="cuda").bfloat16() for _ in range(3))
    cent, _ = _device.centroids(kk, B)
    plan = _device.route(q, cent, B, k)
    for _ in range(3): _device.fwd(q, kk, v, plan, d ** -0.5)
    torch.cuda.synchronize()
    lib.moba_timing_reset(); lib.moba_timing_enable(1)
    for _ in range(10): _device.fwd(q, kk, v, plan, d ** -0.5)
    torch.cuda.synchronize()
    t = _lib.timing_read(); lib.moba_timing_enable(0)
    print((H, N), {s: round(v[0] / max(v[1], 1) * 1e3, 1) for s, v in t.items() if v[1]}, "us")
