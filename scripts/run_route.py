import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11571_b200 import _device
H, N, d, B, k = int(os.environ.get("H", 32)), int(os.environ.get("N", 65536)), 64, 128, 8
mode = int(os.environ.get("MODE", 1))
torch.manual_seed(0)
q, kk = (torch.randn(H, N, d, device="cuda").bfloat16() for _ in range(2))
cent, _ = _device.centroids(kk, B)
for _ in range(3):
    plan = _device.route(q, cent, B, k, mode=mode)
torch.cuda.synchronize()
