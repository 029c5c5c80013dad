"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package from /root/reference/pkg/src (read-only)
and writes one compressed .npz per case into tests/golden/. The fixtures are
committed; nothing on the GPU box reads /root/reference.

Inputs are bf16-representable (torch.randn -> bfloat16 -> float64) so the
GPU path receives exactly the values the reference saw. Each fixture holds
the reference's own outputs of:
  compute_centroids (src/router.py:32), key_conv_forward (src/keyconv.py:70),
  select_topk (src/router.py:49), build_varlen (src/router.py:123),
  moba_attention (src/attention.py:305), moba_backward (src/attention.py:239),
  key_conv_backward (src/keyconv.py:81).
"""

import os
import sys

import numpy as np
import torch

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

# (name, N, B, k, d, conv_width, seed)
CASES = [
    ("c1_fwd_bwd", 2048, 128, 4, 64, 0, 0),      # BASELINE configs[0]
    ("n1024_b128_k8", 1024, 128, 8, 64, 0, 1),   # tests/test_attention.py:85-90 shape
    ("ragged_n500_b64", 500, 64, 3, 64, 0, 2),   # src/verification.py:35 shape
    ("small_n70_b16", 70, 16, 2, 16, 0, 3),      # tests/test_reference.py:150 shape
    ("smalld_n333_b32", 333, 32, 2, 8, 0, 4),
    ("conv3_n512_b64", 512, 64, 4, 64, 3, 5),
    ("conv5_n300_b32", 300, 32, 3, 32, 5, 6),
    ("d128_n768_b128", 768, 128, 4, 128, 0, 7),
    ("saturate_n96_b16", 96, 16, 6, 8, 0, 8),    # dense limit (tests/test_attention.py:76)
    ("c3_like_n1024_b64_k16", 1024, 64, 16, 64, 3, 9),
    ("b8_k1_n200", 200, 8, 1, 16, 0, 10),
]


def bf16_normal(gen, shape):
    return torch.randn(*shape, generator=gen).to(torch.bfloat16).double().numpy()


def f32(x):
    # large float outputs are stored rounded to float32 (fixture size); the
    # oracle is checked against them at float32 resolution
    return np.asarray(x, dtype=np.float32)


def main():
    sys.path.insert(0, REF_SRC)
    import moba  # the reference package

    for name, N, B, k, d, width, seed in CASES:
        gen = torch.Generator().manual_seed(seed)
        Q, K, V, dO = (bf16_normal(gen, (N, d)) for _ in range(4))
        cfg = moba.MobaConfig(block_size_B=B, top_k=k, head_dim_d=d, conv_width=width)
        rec = dict(N=N, B=B, k=k, d=d, width=width,
                   Q=Q.astype(np.float32), K=K.astype(np.float32),
                   V=V.astype(np.float32), dO=dO.astype(np.float32))
        Kc = K
        if width:
            W = moba.random_kernel(width, d, seed=100 + seed).weights
            W = W.astype(np.float32).astype(np.float64)   # fp32-exact weights
            Kc = moba.key_conv_forward(K, moba.ConvKernel(W))
            dKc_probe = dO  # any upstream gradient: reuse dO's values
            dKraw, dW = moba.key_conv_backward(K, moba.ConvKernel(W), dKc_probe)
            rec.update(W=W, Kc=f32(Kc), conv_dK=f32(dKraw), conv_dW=dW)
        cents = moba.compute_centroids(Kc, B)
        idx = moba.select_topk(Q, cents, cfg)
        plan = moba.build_varlen(idx, cents.n_blocks)
        out, plan2 = moba.moba_attention(Q, Kc, V, cfg)
        assert np.array_equal(plan.topk_indices, plan2.topk_indices)
        dQ, dK, dV = moba.moba_backward(Q, Kc, V, out.output, dO, out.logsumexp, plan2, cfg)
        rec.update(centroids=cents.centroids, block_lengths=cents.block_lengths,
                   topk=plan.topk_indices, counts=plan.counts, offsets=plan.offsets,
                   flat=plan.flat_queries, O=f32(out.output), LSE=out.logsumexp,
                   dQ=f32(dQ), dK=f32(dK), dV=f32(dV))
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **rec)
        print(name, "E=", int(plan.counts.sum()))

    # ---- hand cases -----------------------------------------------------
    # tie -> lower index (tests/test_router.py:193-200)
    K = np.tile([1.0, 0.0], (8, 1))
    Q = np.tile([1.0, 0.0], (8, 1))
    cfg = moba.MobaConfig(block_size_B=2, top_k=2, head_dim_d=2)
    idx = moba.select_topk(Q, moba.compute_centroids(K, 2), cfg)
    np.savez_compressed(os.path.join(HERE, "hand_tie.npz"), Q=Q, K=K, B=2, k=2, topk=idx)

    # block-0 rows (tests/test_router.py:149-156)
    rng = np.random.default_rng(1)
    Q = rng.standard_normal((8, 4))
    K = rng.standard_normal((8, 4))
    cfg = moba.MobaConfig(block_size_B=8, top_k=3, head_dim_d=4)
    idx = moba.select_topk(Q, moba.compute_centroids(K, 8), cfg)
    np.savez_compressed(os.path.join(HERE, "hand_block0.npz"), Q=Q, K=K, B=8, k=3, topk=idx)

    # plan without the own block (tests/test_attention.py:234-247)
    gen = torch.Generator().manual_seed(15)
    N, B, d = 64, 16, 8
    Q, K, V, dO = (bf16_normal(gen, (N, d)) for _ in range(4))
    cfg = moba.MobaConfig(block_size_B=B, top_k=1, head_dim_d=d)
    plan = moba.build_varlen(np.zeros((N, 2), dtype=np.int64) - np.array([0, 1]), 4)
    fwd = moba.moba_forward(Q, K, V, plan, cfg)
    dQ, dK, dV = moba.moba_backward(Q, K, V, fwd.output, dO, fwd.logsumexp, plan, cfg)
    np.savez_compressed(os.path.join(HERE, "hand_no_own_block.npz"),
                        Q=Q.astype(np.float32), K=K.astype(np.float32),
                        V=V.astype(np.float32), dO=dO.astype(np.float32),
                        N=N, B=B, k=1, d=d, topk=plan.topk_indices, counts=plan.counts,
                        offsets=plan.offsets, flat=plan.flat_queries,
                        O=fwd.output, LSE=fwd.logsumexp, dQ=dQ, dK=dK, dV=dV)
    print("hand cases written")


if __name__ == "__main__":
    main()
