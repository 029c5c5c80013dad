"""Hybrid MoBA LM parity.

One forward + backward of a toy MobaLM (SWA+RoPE / MoBA+kconv3 alternating,
fp32 parameters and activations) whose MoBA layers run the sm_100a kernels,
against the same model (same weights, same tokens) whose MoBA layers run a
dense masked fp32 PyTorch reference of MoBA attention: bf16 rounding of the
kernel's operands (q, k, v and the conv output K'), the key conv in fp32,
and a block mask from the plan the GPU layer routed with (routing parity is
tested elsewhere; sharing the plan keeps a score tie in one layer from
moving the whole comparison). Both models use the same masked-SDPA
sliding-window layers, so every difference comes from the MoBA operator.
Loss within 2e-2; every parameter gradient within rel-L2 1e-2 (the
north-star tolerance) and max-abs 2e-2.
"""
import copy

import pytest

torch = pytest.importorskip("torch")


pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2511_11571_b200 as mb  # noqa: E402
from paper_2511_11571_b200 import _device, _lib  # noqa: E402
from paper_2511_11571_b200.lm import MobaLM, MobaLMConfig  # noqa: E402


def _rounded(t):
    return t.to(torch.bfloat16).to(torch.float32)


def _conv(k, w):
    """K' = K + silu(sum_l W[l] K_{t-l}), zero left pad (src/keyconv.py:59-78); k [b, h, N, d]."""
    a = torch.zeros_like(k)
    for lag in range(w.shape[0]):
        a[..., lag:, :] = a[..., lag:, :] + w[lag] * k[..., : k.shape[-2] - lag, :]
    return k + a * torch.sigmoid(a)


class Recorder:
    """The kernel operator, recording the plan of every call (routing is
    deterministic: a second routing of the same bf16 inputs is bitwise the
    plan moba_attn used)."""

    def __init__(self):
        self.plans = []

    def __call__(self, q, k, v, B, topk, conv_weight=None, mode="fp32"):
        b, h, N, d = q.shape
        with torch.no_grad():
            qb, kb = (t.to(torch.bfloat16).reshape(-1, N, d).contiguous() for t in (q, k))
            w = None if conv_weight is None else conv_weight.detach().float().contiguous()
            cent, _ = _device.centroids(kb, B, w)
            plan = _device.route(qb, cent, B, topk, _lib.MOBA_ROUTE_TC if mode == "tc" else _lib.MOBA_ROUTE_FP32)
            self.plans.append(plan.topk.clone())
        return mb.moba_attn(q, k, v, B, topk, conv_weight=conv_weight, mode=mode)


class Reference:
    """Dense masked fp32 MoBA attention on the recorded plans (in call order)."""

    def __init__(self, plans):
        self.plans = list(plans)
        self.conv_abs = []          # per MoBA layer: sum over (b, h, t) of |g_t * K_{t-l}| per (l, c)

    def __call__(self, q, k, v, B, topk, conv_weight=None, mode="fp32"):
        b, h, N, d = q.shape
        topk_idx = self.plans.pop(0).view(b, h, N, -1).long()
        qb, kb, vb = _rounded(q), _rounded(k), _rounded(v)
        if conv_weight is not None:
            w = conv_weight.float()
            kc = _conv(kb, w)
            k_in = kb.detach()
            slot = len(self.conv_abs)
            self.conv_abs.append(None)

            def terms(gk, k_in=k_in, w=w.detach(), slot=slot):
                a = torch.zeros_like(k_in)
                for lag in range(w.shape[0]):
                    a[..., lag:, :] += w[lag] * k_in[..., : N - lag, :]
                sg = torch.sigmoid(a)
                g = gk * sg * (1 + a * (1 - sg))
                self.conv_abs[slot] = torch.stack([(g[..., lag:, :] * k_in[..., : N - lag, :]).abs().sum((0, 1, 2))
                                                   for lag in range(w.shape[0])])
            kc.register_hook(terms)
            kb = _rounded(kc)
        blk = torch.arange(N, device=q.device) // B
        sel = (topk_idx[..., :, None, :] == blk[None, None, None, :, None]).any(-1)   # [b, h, N(q), N(k)]
        i = torch.arange(N, device=q.device)
        allowed = sel & (i[None, :] <= i[:, None])
        s = (qb @ kb.transpose(-1, -2)) / d ** 0.5
        s = s.masked_fill(~allowed, float("-inf"))
        return torch.softmax(s, dim=-1) @ vb


def test_hybrid_lm_forward_backward_matches_reference():
    torch.manual_seed(0)
    cfg = MobaLMConfig(vocab=512, hidden=256, heads=4, head_dim=64, intermediate=512, layers=4, block_size=128,
                       top_k=2, conv_width=3, swa_impl="torch", route_mode="tc")
    model = MobaLM(cfg).cuda()
    ref = copy.deepcopy(model)
    tokens = torch.randint(0, cfg.vocab, (2, 1024), device="cuda")
    rec = Recorder()
    for blk in model.blocks:
        blk.attn.moba_fn = rec
    loss = model.loss(tokens)
    loss.backward()
    assert len(rec.plans) == cfg.layers // 2
    reference = Reference(rec.plans)
    for blk in ref.blocks:
        blk.attn.moba_fn = reference
    loss_ref = ref.loss(tokens)
    loss_ref.backward()
    assert abs(float(loss) - float(loss_ref)) <= 2e-2, (float(loss), float(loss_ref))
    report = {}
    conv_abs = iter(reference.conv_abs)
    for (name, p), (_, pr) in zip(model.named_parameters(), ref.named_parameters()):
        assert p.grad is not None and pr.grad is not None, name
        g, r = p.grad.double(), pr.grad.double()
        err = (g - r).abs()
        rel = float((g - r).norm() / r.norm().clamp_min(1e-30))
        report[name] = (float(err.max()), rel)
        if name.endswith("attn.conv"):
            # dW[l, c] = sum over b*h*N = 8192 terms g_t K_{t-l} whose signs
            # cancel; kernel and reference round dK' to bf16 independently
            # (<= 2^-9 per term each), so the derived bound is elementwise
            # 2 * 2^-9 * sum|terms| (2x margin: 2^-7), not a ratio to |dW|
            bound = 2.0 ** -7 * next(conv_abs).double() + 1e-9
            assert bool((err <= bound).all()), (name, float((err - bound).max()))
        else:
            assert report[name][0] <= 2e-2 and rel <= 1e-2, (name, report[name])
    print({k: f"{a:.2e}/{b:.2e}" for k, (a, b) in report.items()})
    assert len(report) == len(list(model.parameters()))
