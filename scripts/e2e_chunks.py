"""e2e (pinned host in/out, moba_fwd_bwd_host) ms per step at the metric
point for several head-chunk counts: python scripts/e2e_chunks.py 8 16 32"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11571_b200 as mb
H, N, d, B, k = (int(x) for x in os.environ.get("CFG", "32,65536,64,128,8").split(","))
g = torch.Generator(device="cuda").manual_seed(0)
pin = [torch.randn(H, N, d, generator=g, device="cuda").bfloat16().cpu().pin_memory() for _ in range(4)]
outs = (torch.empty((H, N, d), dtype=torch.bfloat16).pin_memory(), torch.empty((H, N), dtype=torch.float32).pin_memory(),
        *(torch.empty((H, N, d), dtype=torch.bfloat16).pin_memory() for _ in range(3)))
for nc in [int(a) for a in sys.argv[1:]] or [8, 16, 32]:
    ts = []
    for i in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        mb.moba_fwd_bwd_host(*pin, B, k, n_chunks=nc, out=outs, synchronize=False)
        b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"chunks {nc}: e2e {min(ts[2:]):.2f} ms (median {sorted(ts[2:])[len(ts[2:]) // 2]:.2f})", flush=True)
