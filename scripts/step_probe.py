"""Two eager moba_attn fwd+bwd steps at one shape (for an ncu launch list of
a whole step): python scripts/step_probe.py [H N d B k]"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11571_b200 as mb
H, N, d, B, k = (int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (32, 524288, 64, 128, 8)))
g = torch.Generator(device="cuda").manual_seed(0)
q, kk, v, do = (torch.randn(H, N, d, generator=g, device="cuda").bfloat16().requires_grad_(True) for _ in range(4))
for _ in range(2):
    o = mb.moba_attn(q, kk, v, B, k, mode="tc")
    o.backward(do)
torch.cuda.synchronize()
print("ok")
