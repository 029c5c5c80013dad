"""e2e host-pipeline time vs number of head chunks (pinned host buffers)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11571_b200 as mb
H, N, d, B, k = 16, 8192, 64, 128, 8
pin = [torch.randn(H, N, d).bfloat16().pin_memory() for _ in range(4)]
outs = (torch.empty((H, N, d), dtype=torch.bfloat16).pin_memory(), torch.empty((H, N), dtype=torch.float32).pin_memory(),
        *(torch.empty((H, N, d), dtype=torch.bfloat16).pin_memory() for _ in range(3)))
x = torch.empty(1 << 26, dtype=torch.uint8).pin_memory(); y = torch.empty(1 << 26, dtype=torch.uint8, device="cuda")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3): y.copy_(x, non_blocking=True)
a.record(); y.copy_(x, non_blocking=True); b.record(); torch.cuda.synchronize(); print(f"H2D 64 MB: {64/1024/a.elapsed_time(b)*1e3:.1f} GB/s")
a.record(); x.copy_(y, non_blocking=True); b.record(); torch.cuda.synchronize(); print(f"D2H 64 MB: {64/1024/a.elapsed_time(b)*1e3:.1f} GB/s")
for graphs in (False, True):
  for nc in (2, 4, 8, 16):
    for _ in range(3): mb.moba_fwd_bwd_host(*pin, B, k, n_chunks=nc, mode="tc", out=outs, graphs=graphs)
    ts = []
    for _ in range(5):
        a.record(); mb.moba_fwd_bwd_host(*pin, B, k, n_chunks=nc, mode="tc", out=outs, synchronize=False, graphs=graphs); b.record()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); print(f"graphs {graphs} chunks {nc:2d}: {ts[2]:.3f} ms")
