"""PCIe copy rates on this box: pinned H2D alone, D2H alone, and both at once
on two streams (64 MB each way, the e2e step's volume)."""
import torch
n = 64 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
def h2d():
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
def d2h():
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
def both():
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
for name, fn, nbytes in (("H2D", h2d, n), ("D2H", d2h, n), ("H2D+D2H concurrent", both, 2 * n)):
    ms = timed(fn)
    print(f"{name}: {ms:.3f} ms, {nbytes / ms / 1e6:.1f} GB/s")

# chunked pipeline of copies only (no kernels): 8 chunks, 4 H2D tensors in,
# 5 D2H tensors out per chunk, D2H(c) after H2D(c) — the e2e copy pattern
H, N, d = 16, 8192, 64
hin = [torch.empty(H, N, d, dtype=torch.bfloat16).pin_memory() for _ in range(4)]
hout = [torch.empty(H, N, d, dtype=torch.bfloat16).pin_memory() for _ in range(4)] + [torch.empty(H, N).pin_memory()]
din = [torch.empty(H, N, d, dtype=torch.bfloat16, device="cuda") for _ in range(4)]
dout = [torch.empty(H, N, d, dtype=torch.bfloat16, device="cuda") for _ in range(4)] + [torch.empty(H, N, device="cuda")]
for nc in (4, 8):
    hc = H // nc
    def pipe():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur); s2.wait_stream(cur)
        for c in range(nc):
            h0, h1 = c * hc, (c + 1) * hc
            with torch.cuda.stream(s1):
                for a_, b_ in zip(din, hin): a_[h0:h1].copy_(b_[h0:h1], non_blocking=True)
                ev = torch.cuda.Event(); ev.record(s1)
            with torch.cuda.stream(s2):
                s2.wait_event(ev)
                for a_, b_ in zip(hout, dout): a_[h0:h1].copy_(b_[h0:h1], non_blocking=True)
        cur.wait_stream(s1); cur.wait_stream(s2)
    print(f"copy-only pipeline, {nc} chunks: {timed(pipe):.3f} ms")
