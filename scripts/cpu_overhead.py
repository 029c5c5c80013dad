"""Host-side enqueue time of one moba_attn fwd+bwd step vs its device time."""
import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11571_b200 as mb
H, N, d, B, k = 16, 8192, 64, 128, 8
q, kk, v, do = (torch.randn(H, N, d, device="cuda").bfloat16() for _ in range(4))
qg, kg, vg = (t.clone().requires_grad_(True) for t in (q, kk, v))
def step():
    for t in (qg, kg, vg): t.grad = None
    o = mb.moba_attn(qg, kg, vg, B, k, mode="tc")
    o.backward(do)
for _ in range(5): step()
torch.cuda.synchronize()
big = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
for trial in range(3):
    for _ in range(8): big.zero_()          # ~1 ms of queued GPU work so the host runs ahead
    t0 = time.perf_counter(); step(); t1 = time.perf_counter()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); step(); b.record(); torch.cuda.synchronize()
    print(f"host enqueue {1e3*(t1-t0):.3f} ms   device (no head start) {a.elapsed_time(b):.3f} ms")
