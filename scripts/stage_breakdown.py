"""Per-stage device time (library CUDA-event timers) of one fwd+bwd step for the BASELINE configs."""
import os, sys, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11571_b200 as mb
from paper_2511_11571_b200 import _lib
lib = _lib.load()
CFGS = {
    "C2 h16 N8K d64 B128 k8": (16, 8192, 64, 128, 8, 0),
    "metric b2h16 N64K d64 B128 k8": (32, 65536, 64, 128, 8, 0),
    "C3 h16 N32K d64 B64 k16 conv3": (16, 32768, 64, 64, 16, 3),
    "C4 h16 N64K d128 B128 k8": (16, 65536, 128, 128, 8, 0),
}
only = sys.argv[1:] or list(CFGS)
for name in CFGS:
    if not any(o in name for o in only):
        continue
    H, N, d, B, k, W = CFGS[name]
    torch.manual_seed(0)
    q, kk, v, do = (torch.randn(H, N, d, device="cuda").bfloat16().requires_grad_(True) for _ in range(4))
    w = (torch.rand(W, d, device="cuda") - 0.5).requires_grad_(True) if W else None
    def step():
        for t in (q, kk, v):
            t.grad = None
        o = mb.moba_attn(q, kk, v, B, k, conv_weight=w, mode=os.environ.get("MODE", "tc"))
        o.backward(do)
    try:
        step(); step(); torch.cuda.synchronize()
        lib.moba_timing_reset(); lib.moba_timing_enable(1)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(3): step()
        ev[1].record(); torch.cuda.synchronize()
        t = _lib.timing_read(); lib.moba_timing_enable(0)
        st = {s: round(v_[0] / 3, 3) for s, v_ in t.items() if v_[1]}
        print(f"{name}: step {ev[0].elapsed_time(ev[1]) / 3:.3f} ms  stages(ms) {st}", flush=True)
    except Exception as e:
        print(f"{name}: ERROR {type(e).__name__}: {str(e)[:200]}", flush=True)
    del q, kk, v, do
    torch.cuda.empty_cache()
