"""Route + varlen once per size (for an ncu launch list of the varlen kernels):
python scripts/varlen_probe.py 65536 524288"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11571_b200 import _device, _lib
_lib.load()
for N in [int(a) for a in sys.argv[1:]] or [65536]:
    H, d, B, k = 32, 64, 128, 8
    g = torch.Generator(device="cuda").manual_seed(0)
    q, kk = (torch.randn(H, N, d, generator=g, device="cuda").bfloat16() for _ in range(2))
    cent, _ = _device.centroids(kk, B)
    for _ in range(2):
        plan = _device.route(q, cent, B, k, mode=_lib.MOBA_ROUTE_TC)
    torch.cuda.synchronize()
    print(N, "ok", flush=True)
    del q, kk, cent, plan
    torch.cuda.empty_cache()
