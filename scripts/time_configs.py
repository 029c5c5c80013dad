"""Graph-replayed fwd+bwd step time for the parity configs (no L2 flush):
C2 (16 h x 8K, d64, B128, k8), C3 (16 h x 32K, d64, B64, k16, conv3),
C4 (16 h x 64K, d128, B128, k8) and the 64K metric shape (32 h, d64)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11571_b200 as mb

CFGS = {"C2": (16, 8192, 64, 128, 8, 0), "C3": (16, 32768, 64, 64, 16, 3),
        "C4": (16, 65536, 128, 128, 8, 0), "64K": (32, 65536, 64, 128, 8, 0)}
for name in (sys.argv[1:] or list(CFGS)):
    H, N, d, B, k, conv = CFGS[name]
    torch.manual_seed(0)
    q, kk, v, do = (torch.randn(H, N, d, device="cuda").bfloat16() for _ in range(4))
    w = torch.randn(conv, d, device="cuda") * 0.3 if conv else None
    gs = mb.MobaGraphedStep((H, N, d), B, k, mode="tc", conv_weight=w)
    gs.step(q, kk, v, do)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20 if N <= 8192 else 5
    a.record()
    for _ in range(reps):
        gs.replay()
    b.record()
    torch.cuda.synchronize()
    print(f"{name}: H{H} N{N} d{d} B{B} k{k} conv{conv}: {a.elapsed_time(b) / reps:.3f} ms/step", flush=True)
    del gs
    torch.cuda.empty_cache()
