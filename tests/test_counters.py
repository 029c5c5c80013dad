"""OpCounters parity: the closed forms of
paper_2511_11571_b200/counters.py reproduce the reference's own counter
values (tests/golden/counters.npz, written by tests/golden/make_counters.py
from the reference) — bulk / gathered classification of the Br-row tiles
(src/attention.py:77-86), per-tile score counts (src/router.py:85-88),
centroid traffic (src/router.py:44-45) — including tile knobs that do not
divide B. The CPU test evaluates the closed forms on the reference's plan;
the GPU test runs the package's moba_attention / moba_backward."""
import os

import numpy as np
import pytest
import torch

import paper_2511_11571_b200 as mb
from conftest import GOLDEN
from oracle import moba_oracle as orc
from paper_2511_11571_b200 import _device
from paper_2511_11571_b200.counters import add_backward_counters, add_forward_counters, add_plan_counters
from paper_2511_11571_b200.core import RoutingPlan

G = dict(np.load(os.path.join(GOLDEN, "counters.npz")))
CASES = sorted({k.split("_")[0] for k in G})


def _cfg(p):
    N, B, k, d, Bq, Br, Bc, seed = (int(x) for x in p)
    return N, d, seed, mb.MobaConfig(block_size_B=B, top_k=k, head_dim_d=d, logical_q_block_Bq=Bq,
                                     phys_tile_Br=Br, phys_tile_Bc=Bc)


def _as_dict(arr):
    return dict(zip(("score_flops", "attn_flops", "gathered_elems", "bulk_elems"), (int(x) for x in arr)))


@pytest.mark.parametrize("case", CASES)
def test_closed_forms_match_reference_counters(case):
    N, d, _, cfg = _cfg(G[case + "_params"])
    topk = G[case + "_topk"]
    op = orc.build_varlen(topk, cfg.n_blocks(N))
    t = lambda a: torch.as_tensor(np.asarray(a, dtype=np.int32))[None]
    flat = np.zeros(topk.size, np.int32)
    flat[: len(op.flat_queries)] = op.flat_queries
    plan = RoutingPlan(t(topk), t(op.counts), t(op.offsets), t(flat), None, N, cfg.block_size_B)
    vis = _device.visible_pairs(plan)
    c = mb.OpCounters()
    add_plan_counters(c, 1, N, d, cfg.block_size_B, cfg.phys_tile_Br)
    assert c.as_dict() == _as_dict(G[case + "_plan"])
    c = mb.OpCounters()
    add_forward_counters(c, plan, d, cfg, vis)
    assert c.as_dict() == _as_dict(G[case + "_fwd"])
    c = mb.OpCounters()
    add_backward_counters(c, plan, d, cfg, vis)
    assert c.as_dict() == _as_dict(G[case + "_bwd"])


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_gpu_api_counters_match_reference(case):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    N, d, seed, cfg = _cfg(G[case + "_params"])
    gen = torch.Generator().manual_seed(seed)
    Q, K, V, dO = (torch.randn(N, d, generator=gen).to(torch.bfloat16).double().numpy() for _ in range(4))
    c_att = mb.OpCounters()
    res, plan = mb.moba_attention(Q, K, V, cfg, c_att)
    assert np.array_equal(plan.topk_indices, G[case + "_topk"])
    ref = _as_dict(G[case + "_plan"] + G[case + "_fwd"])
    assert c_att.as_dict() == ref
    c_plan = mb.OpCounters()
    mb.build_plan(Q, K, cfg, c_plan)
    assert c_plan.as_dict() == _as_dict(G[case + "_plan"])
    c_bwd = mb.OpCounters()
    mb.moba_backward(Q, K, V, res.output, dO, res.logsumexp, plan, cfg, c_bwd)
    assert c_bwd.as_dict() == _as_dict(G[case + "_bwd"])
