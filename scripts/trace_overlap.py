"""Forward timeline of CTA 0 (MOBA_FWD_TRACE): per-item softmax intervals of
the two warpgroups, how much of the time both run at once, and the item
period. Needs a timeline build (scripts/README.md, -DMOBA_TIMELINE; the
recording is compiled out of the product library); MOBA_FWD_TRACE_CTA picks
the CTA."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11571_b200 import _device
H, N, d, B, k = (int(x) for x in os.environ.get("CFG", "32,65536,64,128,8").split(","))
torch.manual_seed(0)
q, kk, v = (torch.randn(H, N, d, device="cuda").bfloat16() for _ in range(3))
cent, _ = _device.centroids(kk, B)
plan = _device.route(q, cent, B, k, mode=1)
for _ in range(2): _device.fwd(q, kk, v, plan, d ** -0.5)
torch.cuda.synchronize()
os.environ["MOBA_FWD_TRACE"] = "/tmp/fwd_ov.bin"
_device.fwd(q, kk, v, plan, d ** -0.5)
torch.cuda.synchronize()
t = np.fromfile("/tmp/fwd_ov.bin", dtype=np.int64).reshape(256, 16)
if not t.any():
    sys.exit("empty timeline: build the library with -DMOBA_TIMELINE (scripts/README.md)")
rows = [i for i in range(40, 200) if t[i, 8] and t[i, 9]]
s_ok, p_done = t[rows, 8], t[rows, 9]
busy = np.zeros(int(p_done.max() - s_ok.min()) + 1, dtype=np.int8)
base = s_ok.min()
for a, b, i in zip(s_ok, p_done, rows):
    busy[a - base:b - base] += 1
span = len(busy)
print(f"items {len(rows)}: period {span / len(rows):.0f} clk, softmax {np.median(p_done - s_ok):.0f} clk, "
      f"both WGs busy {np.mean(busy >= 2) * 100:.1f}%, one busy {np.mean(busy == 1) * 100:.1f}%, none {np.mean(busy == 0) * 100:.1f}%")
if any(t[i, 15] for i in rows):
    upto = np.median([t[i, 15] - t[i, 8] for i in rows if t[i, 15]])
    post = np.median([t[i, 9] - t[i, 15] for i in rows if t[i, 15]])
    print(f"softmax split: load + max + p_free wait {upto:.0f}, exp + sums + P store {post:.0f} clk")
