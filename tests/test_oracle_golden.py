"""Pin the CPU oracle (oracle/moba_oracle.py) to the reference's own outputs.

The fixtures in tests/golden/ were produced by running the reference package
(tests/golden/make_golden.py). Integer outputs must match bit-for-bit; float
outputs to float32 storage resolution.
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_names
from oracle import moba_oracle as orc


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def f64(x):
    return np.asarray(x, dtype=np.float64)


@pytest.mark.parametrize("name", golden_names())
def test_oracle_matches_reference_fixture(name):
    g = load(name)
    N, B, k, d, width = (int(g[x]) for x in ("N", "B", "k", "d", "width"))
    Q, K, V, dO = (f64(g[x]) for x in ("Q", "K", "V", "dO"))
    Kc = K
    if width:
        Kc = orc.key_conv_forward(K, g["W"])
        np.testing.assert_allclose(Kc, g["Kc"], rtol=2e-7, atol=2e-7)
        dK_raw, dW = orc.key_conv_backward(K, g["W"], dO)
        np.testing.assert_allclose(dK_raw, g["conv_dK"], rtol=2e-7, atol=2e-7)
        np.testing.assert_allclose(dW, g["conv_dW"], rtol=1e-12, atol=1e-12)
    c, lens = orc.centroids(Kc, B)
    np.testing.assert_allclose(c, g["centroids"], rtol=1e-12, atol=1e-14)
    assert np.array_equal(lens, g["block_lengths"])
    topk = orc.select_topk(Q, c, B, k)
    assert np.array_equal(topk, g["topk"])
    plan = orc.build_varlen(topk, c.shape[0])
    assert np.array_equal(plan.counts, g["counts"])
    assert np.array_equal(plan.offsets, g["offsets"])
    assert np.array_equal(plan.flat_queries, g["flat"])
    orc.validate_plan(plan, N, B)
    assert int(plan.counts.sum()) == orc.plan_entries(N, B, k)
    O, L = orc.forward(Q, Kc, V, plan, B)
    np.testing.assert_allclose(O, g["O"], rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(L, g["LSE"], rtol=1e-12, atol=1e-12)
    dQ, dK, dV = orc.backward(Q, Kc, V, O, dO, L, plan, B)
    for got, ref in ((dQ, g["dQ"]), (dK, g["dK"]), (dV, g["dV"])):
        np.testing.assert_allclose(got, ref, rtol=1e-5, atol=2e-6)


def test_tie_to_lower_index():
    g = load("hand_tie")
    c, _ = orc.centroids(g["K"], int(g["B"]))
    topk = orc.select_topk(g["Q"], c, int(g["B"]), int(g["k"]))
    assert np.array_equal(topk, g["topk"])
    assert [int(x) for x in topk[7] if x >= 0] == [0, 1, 3]   # tests/test_router.py:200


def test_block0_rows():
    g = load("hand_block0")
    c, _ = orc.centroids(g["K"], int(g["B"]))
    topk = orc.select_topk(g["Q"], c, int(g["B"]), int(g["k"]))
    assert np.array_equal(topk, g["topk"])
    assert np.array_equal(topk, np.tile([0, -1, -1, -1], (8, 1)))


def test_plan_without_own_block():
    g = load("hand_no_own_block")
    B = int(g["B"])
    plan = orc.build_varlen(g["topk"], 4)
    assert np.array_equal(plan.flat_queries, g["flat"])
    Q, K, V, dO = (f64(g[x]) for x in ("Q", "K", "V", "dO"))
    O, L = orc.forward(Q, K, V, plan, B)
    np.testing.assert_allclose(O, g["O"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(L, g["LSE"], rtol=1e-12, atol=1e-12)
    dQ, dK, dV = orc.backward(Q, K, V, O, dO, L, plan, B)
    np.testing.assert_allclose(dQ, g["dQ"], atol=1e-12)
    np.testing.assert_allclose(dK, g["dK"], atol=1e-12)
    np.testing.assert_allclose(dV, g["dV"], atol=1e-12)
    assert not dK[B:].any() and not dV[B:].any()


# ---- reference known answers (no fixture needed) -------------------------

def test_centroid_known_answers():
    # tests/test_router.py:127-136
    c, _ = orc.centroids(np.array([[1.0, 0.0], [0.0, 1.0]]), 2)
    assert np.array_equal(c, [[0.5, 0.5]])
    K = np.arange(10, dtype=float).reshape(5, 2)
    c, lens = orc.centroids(K, 2)
    assert lens.tolist() == [2, 2, 1] and np.array_equal(c[2], K[4])


def test_conv_known_answers():
    # tests/test_keyconv.py:17-32
    out = orc.key_conv_forward(np.ones((3, 1)), np.array([[1.0], [0.0], [0.0]]))
    assert np.abs(out - (1.0 + 1.0 / (1.0 + np.exp(-1.0)))).max() <= 1e-12
    silu = lambda x: x / (1.0 + np.exp(-x))
    out = orc.key_conv_forward(np.array([[2.0], [3.0], [5.0]]), np.array([[0.0], [1.0]]))
    np.testing.assert_allclose(out, [[2.0], [3.0 + silu(2.0)], [5.0 + silu(3.0)]], atol=1e-15)


def test_varlen_hand_case():
    # tests/test_router.py:213-217
    plan = orc.build_varlen(np.array([[0], [0], [1]]), 2)
    assert plan.counts.tolist() == [2, 1]
    assert plan.offsets.tolist() == [0, 2]
    assert plan.flat_queries.tolist() == [0, 1, 2]


def test_flop_ratio_gate():
    # tests/test_acceptance.py:187-201: routed/dense MACs at N=8192 in [0.115, 0.135]
    r = orc.visible_pairs(8192, 128, 8) / (8192 * 8192)
    assert 0.115 <= r <= 0.135
    assert abs(r - 0.12408) < 1e-4


@pytest.mark.parametrize("name", ["ragged_n500_b64", "conv3_n512_b64"])
def test_row_and_block_restrictions_match_whole_head_oracle(name):
    """forward_rows / backward_rows_dq / backward_block (used for sampled
    checks at 512K) equal the whole-head oracle on a pinned fixture."""
    g = load(name)
    B = int(g["B"])
    Q, V, dO = (f64(g[x]) for x in ("Q", "V", "dO"))
    K = f64(g["Kc"]) if int(g["width"]) else f64(g["K"])
    plan = orc.OraclePlan(g["topk"], g["counts"], g["offsets"], g["flat"])
    O, L = orc.forward(Q, K, V, plan, B)
    dQ, dK, dV = orc.backward(Q, K, V, O, dO, L, plan, B)
    rows = np.arange(0, Q.shape[0], 7)
    Or, Lr = orc.forward_rows(Q, K, V, rows, g["topk"][rows], B)
    np.testing.assert_allclose(Or, O[rows], atol=1e-12)
    np.testing.assert_allclose(Lr, L[rows], atol=1e-12)
    dq = orc.backward_rows_dq(Q, K, V, O[rows], dO, L[rows], rows, g["topk"][rows], B)
    np.testing.assert_allclose(dq, dQ[rows], atol=1e-12)
    for j in (0, len(g["counts"]) - 1):
        q = orc._block_slice(plan, j)
        dk, dv = orc.backward_block(Q, K, V, dO, j, q, O[q], L[q], B)
        np.testing.assert_allclose(dk, dK[j * B: j * B + len(dk)], atol=1e-12)
        np.testing.assert_allclose(dv, dV[j * B: j * B + len(dv)], atol=1e-12)
