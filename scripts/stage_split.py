"""Per-stage device time (CUDA-event stage timers inside the library) of an
eager fwd+bwd step for the parity configs: python scripts/stage_split.py [C2 C3 C4 64K]."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11571_b200 as mb
from paper_2511_11571_b200 import _lib

CFGS = {"C2": (16, 8192, 64, 128, 8, 0), "C3": (16, 32768, 64, 64, 16, 3),
        "C4": (16, 65536, 128, 128, 8, 0), "64K": (32, 65536, 64, 128, 8, 0),
        "256K": (32, 262144, 64, 128, 8, 0), "512K": (32, 524288, 64, 128, 8, 0)}
lib = _lib.load()
for name in (sys.argv[1:] or list(CFGS)):
    H, N, d, B, k, conv = CFGS[name]
    torch.manual_seed(0)
    q, kk, v, do = (torch.randn(H, N, d, device="cuda").bfloat16().requires_grad_(True) for _ in range(4))
    w = (torch.randn(conv, d, device="cuda") * 0.3).requires_grad_(True) if conv else None
    for it in range(4):
        if it == 1:
            torch.cuda.synchronize()
            lib.moba_timing_reset()
            lib.moba_timing_enable(1)
        o = mb.moba_attn(q, kk, v, B, k, mode="tc", conv_weight=w)
        o.backward(do)
    torch.cuda.synchronize()
    st = _lib.timing_read()
    lib.moba_timing_enable(0)
    parts = {s: tot / 3 for s, (tot, n) in st.items() if n > 0}
    print(f"{name}: " + ", ".join(f"{s} {ms:.3f}" for s, ms in parts.items()) + f"  (sum {sum(parts.values()):.3f} ms)", flush=True)
    del q, kk, v, do, o
    torch.cuda.empty_cache()
