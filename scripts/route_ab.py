"""Router A/B: time moba_route (tc) at several shapes with the library MOBA_LIB
points at, and check the tc plan bitwise against the fp32 router's at 8K/64K."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11571_b200 import _device, _lib
_lib.load()
tag = os.environ.get("MOBA_LIB", "base")
for (H, N, d, B, k, check) in [(32, 8192, 64, 128, 8, True), (32, 65536, 64, 128, 8, True),
                                (32, 524288, 64, 128, 8, False), (16, 65536, 128, 128, 8, False)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    q, kk = (torch.randn(H, N, d, generator=g, device="cuda").bfloat16() for _ in range(2))
    cent, _ = _device.centroids(kk, B)
    ts = []
    for _ in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); p = _device.route(q, cent, B, k, _lib.MOBA_ROUTE_TC); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    msg = ""
    if check:
        r = _device.route(q, cent, B, k, _lib.MOBA_ROUTE_FP32)
        msg = f" bitwise={bool(torch.equal(p.topk, r.topk))}"
    print(f"{tag}: H={H} N={N} d={d} route+varlen {min(ts[1:]):.3f} ms{msg}", flush=True)
    del q, kk, cent, p
    torch.cuda.empty_cache()
