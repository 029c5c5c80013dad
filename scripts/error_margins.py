"""Max-abs / rel-L2 errors of the GPU path vs the f64 oracle for the parity
cases nearest the tolerance (prints the margin left under max-abs 2e-2 /
rel-L2 1e-2): the key-conv autograd case (C3 shape, scaled down) and a
plain d = 64 / d = 128 case."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11571_b200 as mb
from oracle import moba_oracle as orc


def err(g, r):
    g = np.asarray(g, dtype=np.float64)
    return float(np.abs(g - r).max()), float(np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-30))


def case(H, N, d, B, k, W, seed):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    q, kk, v, do = (torch.randn(H, N, d, generator=gen, device="cuda").bfloat16() for _ in range(4))
    w = torch.tensor(orc.random_conv_weights(W, d, seed=7), dtype=torch.float32, device="cuda") if W else None
    for t in (q, kk, v) + ((w,) if W else ()):
        t.requires_grad_(True)
    out, lse = mb.moba_attn(q, kk, v, B, k, conv_weight=w, return_lse=True)
    out.backward(do)
    Qn, Kn, Vn, dOn = (t.detach().double().cpu().numpy() for t in (q, kk, v, do))
    worst = {}
    for h in range(H):
        Kc = orc.key_conv_forward(Kn[h], w.detach().double().cpu().numpy()) if W else Kn[h]
        plan = orc.build_plan(Qn[h], Kc, B, k)
        O, L = orc.forward(Qn[h], Kc, Vn[h], plan, B)
        rQ, rKc, rV = orc.backward(Qn[h], Kc, Vn[h], O, dOn[h], L, plan, B)
        rK = orc.key_conv_backward(Kn[h], w.detach().double().cpu().numpy(), rKc)[0] if W else rKc
        for name, g, r in (("O", out[h].detach().float().cpu().numpy(), O), ("dQ", q.grad[h].float().cpu().numpy(), rQ),
                           ("dK", kk.grad[h].float().cpu().numpy(), rK), ("dV", v.grad[h].float().cpu().numpy(), rV)):
            e = err(g, r)
            worst[name] = tuple(max(a, b) for a, b in zip(worst.get(name, (0.0, 0.0)), e))
    print(f"H={H} N={N} d={d} B={B} k={k} conv={W}: " +
          ", ".join(f"{n} max-abs {a:.2e} rel {r:.2e}" for n, (a, r) in worst.items()), flush=True)


if __name__ == "__main__":
    torch.cuda.set_device(0)
    case(2, 2048, 64, 64, 16, 3, 5)
    case(2, 4096, 64, 128, 8, 0, 11)
    case(2, 4096, 128, 128, 8, 0, 12)
