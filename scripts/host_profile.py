"""Host-side cost of each stage call of one eager fwd+bwd step (no device sync in between)."""
import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11571_b200 import _device
H, N, d, B, k = 16, 8192, 64, 128, 8
q, kk, v, do = (torch.randn(H, N, d, device="cuda").bfloat16() for _ in range(4))
big = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
def run(times):
    t = time.perf_counter
    a = t(); cent, ku = _device.centroids(kk, B); b = t(); times["centroids"] += b - a
    a = t(); plan = _device.route(q, cent, B, k, mode=1); b = t(); times["route"] += b - a
    a = t(); o, lse = _device.fwd(q, kk, v, plan, d ** -0.5); b = t(); times["fwd"] += b - a
    a = t(); _device.bwd(q, kk, v, o, do, lse, plan, d ** -0.5, deterministic=False); b = t(); times["bwd"] += b - a
times = {k_: 0.0 for k_ in ("centroids", "route", "fwd", "bwd")}
for _ in range(3): run(dict(times))
torch.cuda.synchronize()
for _ in range(10):
    for _ in range(4): big.zero_()      # keep the GPU busy so the host never waits
    run(times)
    torch.cuda.synchronize()
print({k_: round(v_ / 10 * 1e6, 1) for k_, v_ in times.items()}, "us host per call")
