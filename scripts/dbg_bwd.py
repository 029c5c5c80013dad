import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11571_b200 as mb
from paper_2511_11571_b200 import _device
torch.manual_seed(0)
for (H, N, d, B, k) in [(1, 2048, 64, 128, 4), (1, 512, 64, 128, 2), (2, 1024, 128, 128, 4)]:
    q, kk, v, do = (torch.randn(H, N, d, device="cuda").bfloat16() for _ in range(4))
    cent, _ = _device.centroids(kk, B)
    plan = _device.route(q, cent, B, k)
    o, lse = _device.fwd(q, kk, v, plan, d ** -0.5)
    res = {}
    for impl in ("mma", "tc"):
        os.environ["MOBA_BWD_IMPL"] = impl
        for det in (False, True):
            res[(impl, det)] = [t.float() for t in _device.bwd(q, kk, v, o, do, lse, plan, d ** -0.5, deterministic=det)]
    ref = res[("mma", False)]
    for key, val in res.items():
        errs = [float((a - b).abs().max()) for a, b in zip(val, ref)]
        print((H, N, d, B, k), key, "dQ %.3e dK %.3e dV %.3e" % tuple(errs))
    dq_err = (res[("tc", False)][0] - ref[0]).abs().amax(dim=-1)[0]
    bad = torch.nonzero(dq_err > 0.05).flatten()
    print("  bad dQ rows:", bad.numel(), bad[:20].tolist())
    dk_err = (res[("tc", False)][1] - ref[1]).abs().amax(dim=-1)[0]
    bad = torch.nonzero(dk_err > 0.05).flatten()
    print("  bad dK rows:", bad.numel(), bad[:20].tolist(), "  (row % 128):", sorted(set((bad % 128).tolist()))[:40])
