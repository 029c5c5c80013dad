"""Tile statistics of a routing plan (how many 128-row tiles the forward /
backward run, how full they are): python scripts/tile_stats.py [H N d B k]."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11571_b200 import _device
H, N, d, B, k = (int(x) for x in (sys.argv[1:] or "32 65536 64 128 8".split()))
torch.manual_seed(0)
q, kk = (torch.randn(H, N, d, device="cuda").bfloat16() for _ in range(2))
cent, _ = _device.centroids(kk, B)
plan = _device.route(q, cent, B, k, mode=1)
c = plan.counts_d.long()
tiles = (c + 127) // 128
rows = int(c.sum())
nt = int(tiles.sum())
print(f"H={H} N={N} B={B} k={k}: routed rows {rows}, tiles {nt} (fill {rows / (128 * nt):.3f}), "
      f"tiles per SM {nt / 148:.1f}, items {int((c > 0).sum())}")
nb = c.shape[1]
for lo, hi in ((0, nb // 8), (nb // 8, nb // 2), (nb // 2, nb)):
    cc = c[:, lo:hi]
    print(f"  blocks [{lo},{hi}): mean count {float(cc.float().mean()):.0f}, tiles {int(((cc + 127) // 128).sum())}")
hist = torch.bincount(tiles.flatten())
print("  items by tile count:", {i: int(v) for i, v in enumerate(hist.tolist()) if v})
