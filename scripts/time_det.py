"""fwd+bwd step time: parallel vs deterministic dQ schedule (C2 and 64K shapes)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11571_b200 as mb
for (H, N) in ((16, 8192), (32, 65536)):
    q, kk, v, do = (torch.randn(H, N, 64, device="cuda").bfloat16() for _ in range(4))
    for det in (False, True):
        gs = mb.MobaGraphedStep((H, N, 64), 128, 8, mode="tc", deterministic=det)
        gs.step(q, kk, v, do)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5): gs.replay()
        b.record(); torch.cuda.synchronize()
        print(f"H{H} N{N} deterministic={det}: {a.elapsed_time(b) / 5:.3f} ms/step", flush=True)
        del gs
        torch.cuda.empty_cache()
