"""Run the four stages eagerly with a sync after each (locates a failing kernel)."""
import os, sys, torch
sys.path.insert(0, "/root/repo")
from paper_2511_11571_b200 import _device
H, N, d, B, k = 16, 65536, 128, 128, 8
torch.manual_seed(0)
H, N, d = (int(x) for x in os.environ.get("SHAPE", "16,65536,128").split(","))
mk = torch.zeros if os.environ.get("ZERO") else torch.randn
q, kk, v, do = (mk(H, N, d, device="cuda").bfloat16() for _ in range(4))
cent, _ = _device.centroids(kk, B); torch.cuda.synchronize(); print("centroids ok", flush=True)
plan = _device.route(q, cent, B, k, mode=1); torch.cuda.synchronize(); print("route ok", flush=True)
o, lse = _device.fwd(q, kk, v, plan, d ** -0.5); torch.cuda.synchronize(); print("fwd ok", flush=True)
r = _device.bwd(q, kk, v, o, do, lse, plan, d ** -0.5, deterministic=False); torch.cuda.synchronize(); print("bwd ok", flush=True)
