import os, sys, torch
sys.path.insert(0, "/root/repo")
import paper_2511_11571_b200 as mb
from paper_2511_11571_b200.attention import moba_attn
H, N, d = (int(x) for x in os.environ.get("SHAPE", "16,65536,128").split(","))
torch.manual_seed(0)
q, kk, v, do = (torch.randn(H, N, d, device="cuda").bfloat16() for _ in range(4))
for mode in ("tc",):
    qq, k2, v2 = (t.clone().requires_grad_(True) for t in (q, kk, v))
    o = moba_attn(qq, k2, v2, 128, 8, mode=mode)
    torch.cuda.synchronize(); print("eager fwd ok", flush=True)
    o.backward(do); torch.cuda.synchronize(); print("eager bwd ok", flush=True)
z = [torch.zeros_like(q).requires_grad_(True) for _ in range(3)]
o = moba_attn(z[0], z[1], z[2], 128, 8, mode="tc"); o.backward(torch.zeros_like(do)); torch.cuda.synchronize(); print("eager zeros ok", flush=True)
gs = mb.MobaGraphedStep((H, N, d), 128, 8, mode="tc", warmup=int(os.environ.get("WARM", "2")))
torch.cuda.synchronize(); print("captured", gs.launches_per_step, flush=True)
gs.replay(); torch.cuda.synchronize(); print("replay zeros ok", flush=True)
gs.step(q, kk, v, do); torch.cuda.synchronize(); print("replay random ok", flush=True)
