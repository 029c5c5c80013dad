"""C5 (BASELINE.json configs[4]): training step of the paper's 340M-class
hybrid MoBA LM (24 layers, SWA-256+RoPE / MoBA B=128 k=8 alternating, d=64),
random init, synthetic tokens. Prints one JSON line: tokens/s and model
TFLOP/s of the full step (forward, loss, backward, AdamW)."""
import argparse, json, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11571_b200.lm import MobaLM, MobaLMConfig, model_flops_per_token, train_step

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=65536)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--layers", type=int, default=24)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--conv", type=int, default=0)
args = ap.parse_args()
torch.manual_seed(0)
cfg = MobaLMConfig(layers=args.layers, conv_width=args.conv)
model = MobaLM(cfg).cuda().to(torch.bfloat16)
opt = torch.optim.AdamW(model.parameters(), lr=1e-4, fused=True)
tokens = torch.randint(0, cfg.vocab, (args.batch, args.seq), device="cuda")
for _ in range(args.warmup):
    train_step(model, opt, tokens)
torch.cuda.synchronize()
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
losses = []
for a, b in evs:
    a.record(); losses.append(train_step(model, opt, tokens)); b.record()
torch.cuda.synchronize()
ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
ntok = args.batch * args.seq
fpt = model_flops_per_token(cfg, args.seq)
print(json.dumps({"workload": f"configs[4]: {cfg.layers}-layer hybrid MoBA LM ({model.n_params() / 1e6:.0f}M params), "
                  f"batch {args.batch} x N={args.seq}, B={cfg.block_size}, k={cfg.top_k}, conv={cfg.conv_width}; "
                  "step = fwd + loss + bwd + AdamW, bf16, random init, synthetic tokens",
                  "ms_per_step": ms, "tokens_per_s": ntok / (ms / 1e3),
                  "model_tflops": fpt * ntok / (ms / 1e3) / 1e12,
                  "loss": [float(l) for l in losses],
                  "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9}))
