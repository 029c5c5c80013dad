"""Host-side logic that needs no GPU: config validation, error classes,
API guards (mirrors tests/test_core.py:127-151 of the reference)."""
import numpy as np
import pytest

import paper_2511_11571_b200 as mb
from paper_2511_11571_b200.router import infer_block_size


def test_config_defaults_and_validation():
    cfg = mb.MobaConfig(block_size_B=128, top_k=8, head_dim_d=64)
    assert cfg.phys_tile_Br == 64 and cfg.phys_tile_Bc == 64 and cfg.logical_q_block_Bq == 512
    assert cfg.n_blocks(8192) == 64 and cfg.n_blocks(8193) == 65
    assert mb.MobaConfig(block_size_B=16, top_k=1, head_dim_d=4).phys_tile_Bc == 16
    for bad in (dict(block_size_B=0, top_k=1, head_dim_d=4), dict(block_size_B=4, top_k=0, head_dim_d=4),
                dict(block_size_B=4, top_k=1, head_dim_d=4, conv_width=4),
                dict(block_size_B=4, top_k=1, head_dim_d=4, phys_tile_Bc=5),
                dict(block_size_B=4, top_k=1, head_dim_d=4, logical_q_block_Bq=0)):
        with pytest.raises(mb.ConfigError):
            mb.MobaConfig(**bad)


def test_error_hierarchy():
    for e in (mb.ShapeError, mb.ConfigError, mb.PlanValidationError, mb.FormatError, mb.LengthError):
        assert issubclass(e, mb.MobaError)


def test_counters_merge():
    a = mb.OpCounters(1, 2, 3, 4)
    b = mb.OpCounters(10, 20, 30, 40)
    a.merge(b)
    assert a.as_dict() == {"score_flops": 11, "attn_flops": 22, "gathered_elems": 33, "bulk_elems": 44}
    a.reset()
    assert a.as_dict() == {"score_flops": 0, "attn_flops": 0, "gathered_elems": 0, "bulk_elems": 0}


def test_threads_cap(monkeypatch):
    monkeypatch.setenv("MOBA_THREADS", "2")
    assert mb.resolve_threads(8) == 2
    assert mb.resolve_threads(None) == 2


def test_causal_false_and_shape_guards_raise_before_device():
    import torch
    q = torch.zeros(2, 64, 8)
    with pytest.raises(mb.ConfigError):
        mb.moba_attn(q, q, q, 16, 2, causal=False)
    with pytest.raises(mb.ShapeError):
        mb.moba_attention(np.zeros((4, 2, 8)), np.zeros((4, 2, 8)), np.zeros((4, 2, 8)),
                          mb.MobaConfig(block_size_B=4, top_k=1, head_dim_d=8))
    with pytest.raises(mb.ShapeError):
        mb.moba_attention(np.zeros((8, 4)), np.zeros((8, 4)), np.zeros((9, 4)),
                          mb.MobaConfig(block_size_B=4, top_k=1, head_dim_d=4))


def test_conv_kernel_validation():
    with pytest.raises(mb.ShapeError):
        mb.ConvKernel(np.zeros(3))
    with pytest.raises(mb.ShapeError):
        mb.ConvKernel(np.array([[np.inf, 0.0]]))
    assert mb.random_kernel(3, 8, seed=1).width == 3
    w = mb.random_kernel(5, 4, seed=2).weights
    assert np.all(np.abs(w) <= 1 / np.sqrt(5))


def test_infer_block_size():
    assert infer_block_size(64, 4) == 16
    assert infer_block_size(70, 5) == 14
    assert -(-70 // infer_block_size(70, 5)) == 5
    with pytest.raises(mb.PlanValidationError):
        infer_block_size(10, 0)
