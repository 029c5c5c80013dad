"""Per-tile timeline of CTA 0 of the d = 128 backward kernel (clock64, MOBA_TRACE)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11571_b200 import _device
H, N, d, B, k = (int(x) for x in os.environ.get("CFG", "16,65536,128,128,8").split(","))
torch.manual_seed(0)
q, kk, v, do = (torch.randn(H, N, d, device="cuda").bfloat16() for _ in range(4))
cent, _ = _device.centroids(kk, B)
plan = _device.route(q, cent, B, k, mode=1)
o, lse = _device.fwd(q, kk, v, plan, d ** -0.5)
for _ in range(2): _device.bwd(q, kk, v, o, do, lse, plan, d ** -0.5, deterministic=False)
torch.cuda.synchronize()
path = "/tmp/bwd128_trace.bin"
os.environ["MOBA_TRACE"] = path
_device.bwd(q, kk, v, o, do, lse, plan, d ** -0.5, deterministic=False)
torch.cuda.synchronize()
t = np.fromfile(path, dtype=np.int64).reshape(64, 16)
t0 = t[t > 0].min()
names = ["P:qe_ok", "P:issued", "M:qd_ok", "M:s_iss", "M:pa_ok", "M:p_ok", "S:s_ok", "S:dp_ok", "S:done",
         "E:dq_ok", "E:done"]
print("g   " + " ".join(f"{n:>10s}" for n in names))
rows = [i for i in range(64) if t[i].any()]
for i in rows[:int(os.environ.get("ROWS", 16))]:
    print(f"{i:3d} " + " ".join(f"{(t[i, e] - t0) if t[i, e] else -1:10d}" for e in range(11)))
span = t[rows].max() - t0
print(f"tiles {len(rows)}, span {span} cycles, {span / max(len(rows), 1):.0f} cycles/tile")
