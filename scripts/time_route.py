"""Routing + varlen stage times (library CUDA-event timers)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11571_b200 import _device, _lib
lib = _lib.load()
CFGS = [(16, 8192, 64, 128, 8), (32, 65536, 64, 128, 8), (16, 32768, 64, 64, 16), (16, 65536, 128, 128, 8)]
for (H, N, d, B, k) in CFGS:
    torch.manual_seed(0)
    q, kk = (torch.randn(H, N, d, device="cuda").bfloat16() for _ in range(2))
    cent, _ = _device.centroids(kk, B)
    for mode in (1, 0):
        ref = _device.route(q, cent, B, k, mode=mode)
        torch.cuda.synchronize()
        lib.moba_timing_reset(); lib.moba_timing_enable(1)
        for _ in range(5): plan = _device.route(q, cent, B, k, mode=mode)
        torch.cuda.synchronize()
        t = _lib.timing_read(); lib.moba_timing_enable(0)
        same = bool(torch.equal(plan.flat_d, ref.flat_d) and torch.equal(plan.row_pos, ref.row_pos))
        print(f"H{H} N{N} d{d} B{B} k{k} mode={'tc' if mode else 'fp32'}",
              {s: round(v_[0] / max(v_[1], 1) * 1e3, 1) for s, v_ in t.items() if v_[1]}, "us  deterministic:", same, flush=True)
    del q, kk, cent
    torch.cuda.empty_cache()
