import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2511_11571_b200 import _device
H, N, d, B, k = 32, 65536, 64, 128, 8
torch.manual_seed(0)
q, kk, v = (torch.randn(H, N, d, device="cuda").bfloat16() for _ in range(3))
cent, _ = _device.centroids(kk, B)
plan = _device.route(q, cent, B, k, mode=1)
for _ in range(2): _device.fwd(q, kk, v, plan, d ** -0.5)
torch.cuda.synchronize()
os.environ["MOBA_FWD_TRACE"] = "/tmp/fwd_cta.bin"
_device.fwd(q, kk, v, plan, d ** -0.5); torch.cuda.synchronize()
t = np.fromfile("/tmp/fwd_cta.bin", dtype=np.int64)
end, nl, st = t[4096:4096+148], t[4096+256:4096+256+148], t[4096+512:4096+512+148]
t0 = st.min()
e = (end - t0) / 1e3; s0 = (st - t0) / 1e3
print("start us: max %.1f" % s0.max())
print("end us: min %.1f median %.1f max %.1f" % (e.min(), np.median(e), e.max()))
print("items per CTA", nl.min(), nl.max())
order = np.argsort(e)
print("fastest CTAs", order[:8], e[order[:8]].round(0))
print("slowest CTAs", order[-8:], e[order[-8:]].round(0))
print("end by CTA index (every 10th):", [round(x) for x in e[::10]])
