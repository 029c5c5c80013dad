"""Forward stage times (library CUDA-event timers) per fwd implementation.
usage: python scripts/time_fwd.py [impl ...]   (impl: t = ping-pong TS kernel, w = warp-specialised SS, s = simple tc)"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11571_b200 import _device, _lib
lib = _lib.load()
impls = sys.argv[1:] or ["t", "w"]
CFGS = [(16, 8192, 64, 128, 8), (32, 65536, 64, 128, 8), (16, 32768, 64, 64, 16), (16, 65536, 128, 128, 8)]
for (H, N, d, B, k) in CFGS:
    torch.manual_seed(0)
    q, kk, v = (torch.randn(H, N, d, device="cuda").bfloat16() for _ in range(3))
    cent, _ = _device.centroids(kk, B)
    plan = _device.route(q, cent, B, k)
    ref = None
    for impl in impls:
        os.environ["MOBA_FWD_IMPL"] = impl
        for _ in range(3): o, l = _device.fwd(q, kk, v, plan, d ** -0.5)
        torch.cuda.synchronize()
        if ref is None:
            ref = (o.float(), l)
            err = 0.0
        else:
            err = max((o.float() - ref[0]).abs().max().item(), (l - ref[1]).abs().max().item())
        lib.moba_timing_reset(); lib.moba_timing_enable(1)
        for _ in range(10): _device.fwd(q, kk, v, plan, d ** -0.5)
        torch.cuda.synchronize()
        t = _lib.timing_read(); lib.moba_timing_enable(0)
        print(f"H{H} N{N} d{d} B{B} k{k} impl={impl}", {s: round(v_[0] / max(v_[1], 1) * 1e3, 1) for s, v_ in t.items() if v_[1]},
              f"us  max|diff vs {impls[0]}| {err:.2e}", flush=True)
    del q, kk, v, plan
    torch.cuda.empty_cache()
