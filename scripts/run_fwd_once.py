"""Run one config's forward a few times (driver for ncu captures).
env: CFG=H,N,d,B,k (default 16,8192,64,128,8), MOBA_FWD_IMPL."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11571_b200 import _device
H, N, d, B, k = (int(x) for x in os.environ.get("CFG", "16,8192,64,128,8").split(","))
torch.manual_seed(0)
q, kk, v = (torch.randn(H, N, d, device="cuda").bfloat16() for _ in range(3))
cent, _ = _device.centroids(kk, B)
plan = _device.route(q, cent, B, k, mode=1)
for _ in range(4):
    _device.fwd(q, kk, v, plan, d ** -0.5)
torch.cuda.synchronize()
