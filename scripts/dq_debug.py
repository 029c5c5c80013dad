"""Compare dQ of the parallel (atomic) and deterministic backward schedules row by row."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11571_b200 import _device
H, N, d, B, k = (int(x) for x in os.environ.get("CFG", "2,200,64,8,1").split(","))
torch.manual_seed(0)
q, kk, v, do = (torch.randn(H, N, d, device="cuda").bfloat16() for _ in range(4))
cent, _ = _device.centroids(kk, B)
plan = _device.route(q, cent, B, k, mode=0)
o, lse = _device.fwd(q, kk, v, plan, d ** -0.5)
a = _device.bwd(q, kk, v, o, do, lse, plan, d ** -0.5, deterministic=False)[0].float()
b = _device.bwd(q, kk, v, o, do, lse, plan, d ** -0.5, deterministic=True)[0].float()
err = (a - b).abs().amax(-1)
print("max err", err.max().item(), "rows bad", int((err > 1e-2).sum()), "of", H * N)
bad = (err > 1e-2).nonzero()[:10].tolist()
print("first bad (h, row):", bad)
for h, r in bad[:3]:
    print(h, r, a[h, r, :6].tolist(), b[h, r, :6].tolist())
