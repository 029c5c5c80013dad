import os, sys, ctypes, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MOBA_TRACE"] = "1"
from paper_2511_11571_b200 import _device, _lib
lib = _lib.load()
H, N, d, B, k = 16, 8192, 64, 128, 8
torch.manual_seed(0)
q, kk, v, do = (torch.randn(H, N, d, device="cuda").bfloat16() for _ in range(4))
cent, _ = _device.centroids(kk, B)
plan = _device.route(q, cent, B, k)
o, lse = _device.fwd(q, kk, v, plan, d ** -0.5)
for _ in range(3): _device.bwd(q, kk, v, o, do, lse, plan, d ** -0.5, deterministic=False)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (64 * 16))()
lib.moba_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
lib.moba_debug_trace(ctypes.addressof(buf), 64 * 16)
a = np.array(buf).reshape(64, 16)
t0 = a[0, 0]
names = ["P:qd_empty", "P:arrive", "M:qd_full", "M:s_empty", "M:p_full", "M:dq_empty", "S:s_full", "S:p_empty", "S:done", "Q:dq_full", "Q:done"]
print("tile " + " ".join(n.rjust(10) for n in names))
for g in range(24):
    print(str(g).rjust(4), " ".join(str(int(a[g, i] - t0) if a[g, i] else "-").rjust(10) for i in range(11)))
