import os, sys, torch
sys.path.insert(0, "/root/repo")
from paper_2511_11571_b200 import _device
H, N, d, B, k = 16, 8192, 64, 128, 8
torch.manual_seed(0)
q, kk = (torch.randn(H, N, d, device="cuda").bfloat16() for _ in range(2))
cent, _ = _device.centroids(kk, B)
plan = _device.route(q, cent, B, k, mode=1)
import numpy as np; c = torch.as_tensor(np.asarray(plan.counts)).long()
print("pairs", int(c.sum()), "tiles", int(((c + 127) // 128).sum()), "items", c.numel(), "max tiles/item", int(((c+127)//128).max()))
