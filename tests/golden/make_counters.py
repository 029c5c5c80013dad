"""Golden OpCounters from the REFERENCE (run in the build container):

    python tests/golden/make_counters.py

For each case it runs the reference's build_plan, moba_forward (via
moba_attention) and moba_backward with an OpCounters object
(src/core.py:193-226; increments at src/router.py:44-45, :85-88 and
src/attention.py:77-86, :113-141, :204-236, :265-300) on bf16-representable
inputs and stores the inputs' seed, the plan and the four counters of each
call in tests/golden/counters.npz. Cases vary the tile knobs (Bq, Br, Bc),
including Br / Bc that do not divide B, so the bulk / gathered
classification and the per-tile score counts are exercised.
"""

import os
import sys

import numpy as np
import torch

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

# (N, B, k, d, Bq, Br, Bc, seed)
CASES = [
    (1000, 64, 3, 32, 512, None, None, 40),
    (1536, 128, 4, 64, 256, 48, 40, 41),
    (700, 32, 5, 16, 128, 24, 32, 42),
    (2048, 128, 8, 64, 512, 64, 64, 43),
    (333, 16, 2, 8, 64, 7, 5, 44),
]


def main():
    sys.path.insert(0, REF_SRC)
    import moba
    out = {}
    for c, (N, B, k, d, Bq, Br, Bc, seed) in enumerate(CASES):
        gen = torch.Generator().manual_seed(seed)
        Q, K, V, dO = (torch.randn(N, d, generator=gen).to(torch.bfloat16).double().numpy() for _ in range(4))
        cfg = moba.MobaConfig(block_size_B=B, top_k=k, head_dim_d=d, logical_q_block_Bq=Bq,
                              phys_tile_Br=Br, phys_tile_Bc=Bc)
        c_plan, c_fwd, c_bwd = moba.OpCounters(), moba.OpCounters(), moba.OpCounters()
        plan = moba.build_plan(Q, K, cfg, c_plan)
        res = moba.moba_forward(Q, K, V, plan, cfg, c_fwd)
        moba.moba_backward(Q, K, V, res.output, dO, res.logsumexp, plan, cfg, c_bwd)
        out[f"case{c}_params"] = np.array([N, B, k, d, Bq, cfg.phys_tile_Br, cfg.phys_tile_Bc, seed], np.int64)
        out[f"case{c}_topk"] = plan.topk_indices.astype(np.int32)
        for tag, cnt in (("plan", c_plan), ("fwd", c_fwd), ("bwd", c_bwd)):
            out[f"case{c}_{tag}"] = np.array([cnt.score_flops, cnt.attn_flops, cnt.gathered_elems, cnt.bulk_elems],
                                             np.int64)
        print(c, N, B, k, d, Bq, cfg.phys_tile_Br, cfg.phys_tile_Bc, out[f"case{c}_plan"], out[f"case{c}_fwd"],
              out[f"case{c}_bwd"])
    np.savez_compressed(os.path.join(HERE, "counters.npz"), **out)


if __name__ == "__main__":
    main()
