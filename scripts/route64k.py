import os, sys, torch
sys.path.insert(0, "/root/repo")
from paper_2511_11571_b200 import _device
H, N, d, B, k = 32, 65536, 64, 128, 8
torch.manual_seed(0)
q, kk = (torch.randn(H, N, d, device="cuda").bfloat16() for _ in range(2))
cent, _ = _device.centroids(kk, B)
for _ in range(2):
    plan = _device.route(q, cent, B, k, mode=1)
torch.cuda.synchronize()
