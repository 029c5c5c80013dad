"""Route-stage probe: time moba_route at one shape (for ncu: one launch of each kernel)."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11571_b200 import _device, _lib
H, N, d, B, k = (int(x) for x in sys.argv[1:6])
mode = sys.argv[6] if len(sys.argv) > 6 else "tc"
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 3
gen = torch.Generator(device="cuda").manual_seed(0)
q, kk = (torch.randn(H, N, d, generator=gen, device="cuda").bfloat16() for _ in range(2))
cent, _ = _device.centroids(kk, B)
m = _lib.MOBA_ROUTE_TC if mode == "tc" else _lib.MOBA_ROUTE_FP32
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); p = _device.route(q, cent, B, k, m); b.record(); torch.cuda.synchronize()
    print(f"route {mode} H={H} N={N} d={d}: {a.elapsed_time(b):.3f} ms", flush=True)
