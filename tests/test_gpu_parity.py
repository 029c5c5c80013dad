"""GPU parity: the CUDA path against the reference fixtures and the oracle.

Runs on a B200 (`pytest -m gpu`). Every call goes through the package's
reference-shaped API, i.e. through libmoba_b200.so's C ABI.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import GOLDEN, golden_names
from helpers import assert_close, bf16_round, unexcused_routing_rows
from oracle import moba_oracle as orc

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2511_11571_b200 as mb  # noqa: E402


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def f64(x):
    return np.asarray(x, dtype=np.float64)


def cfg_of(g):
    return mb.MobaConfig(block_size_B=int(g["B"]), top_k=int(g["k"]), head_dim_d=int(g["d"]),
                         conv_width=int(g["width"]))


@pytest.mark.parametrize("name", golden_names())
def test_centroids_and_conv_vs_reference(name):
    g = load(name)
    B, width = int(g["B"]), int(g["width"])
    K = f64(g["K"])
    if width:
        kern = mb.ConvKernel(g["W"])
        Kc = mb.key_conv_forward(K, kern)
        # K' is returned from its bf16 kernel copy: round-to-nearest bf16 is
        # within 2^-9 relative, so the bound is elementwise 2^-8 |K'| (2x
        # margin) + 1e-6 for the fp32 conv arithmetic
        err = np.abs(np.asarray(Kc, np.float64) - g["Kc"])
        assert np.all(err <= 2.0 ** -8 * np.abs(g["Kc"]) + 1e-6), float((err - 2.0 ** -8 * np.abs(g["Kc"])).max())
        cents = mb.compute_centroids(K, B)  # raw-K centroids path
        ref_c, _ = orc.centroids(K, B)
        np.testing.assert_allclose(cents.centroids, ref_c, rtol=1e-5, atol=1e-6)
    else:
        cents = mb.compute_centroids(K, B)
        np.testing.assert_allclose(cents.centroids, g["centroids"], rtol=1e-5, atol=1e-6)
        assert np.array_equal(cents.block_lengths, g["block_lengths"])


@pytest.mark.parametrize("name", golden_names())
def test_routing_vs_reference(name):
    g = load(name)
    B, k, width = int(g["B"]), int(g["k"]), int(g["width"])
    cfg = cfg_of(g)
    Q, K = f64(g["Q"]), f64(g["K"])
    if width:
        # route on the fused conv path: centroids of the fp32 K' (moba_attn)
        qt = torch.tensor(g["Q"]).cuda().bfloat16()[None]
        kt = torch.tensor(g["K"]).cuda().bfloat16()[None]
        w = torch.tensor(g["W"], dtype=torch.float32).cuda()
        from paper_2511_11571_b200 import _device
        dp = _device.padded_dim(int(g["d"]))
        pad = lambda t: torch.nn.functional.pad(t, (0, dp - t.shape[-1]))
        cent, _ = _device.centroids(pad(kt).contiguous(), B, pad(w).contiguous())
        plan = _device.route(pad(qt).contiguous(), cent, B, k)
        topk = plan.topk_indices
        ref_cents = g["centroids"]
    else:
        plan = mb.build_plan(Q, K, cfg)
        topk = plan.topk_indices
        ref_cents = g["centroids"]
    bad, ndiff = unexcused_routing_rows(Q, ref_cents, topk, g["topk"], B, k)
    assert not bad, f"{len(bad)} rows differ beyond ties (of {ndiff} differing rows): {bad[:10]}"
    if ndiff == 0:
        assert np.array_equal(plan.counts, g["counts"])
        assert np.array_equal(plan.offsets, g["offsets"])
        assert np.array_equal(plan.flat_queries, g["flat"])
    # invariants always
    orc.validate_plan(orc.OraclePlan(topk, plan.counts, plan.offsets, plan.flat_queries), int(g["N"]), B)


@pytest.mark.parametrize("name", golden_names())
@pytest.mark.parametrize("schedule", ["deterministic", "parallel"])
def test_attention_on_reference_plan(name, schedule):
    """Forward + backward on the reference's own plan vs its outputs."""
    g = load(name)
    cfg = cfg_of(g)
    Q, V, dO = f64(g["Q"]), f64(g["V"]), f64(g["dO"])
    Kc = f64(g["Kc"]) if int(g["width"]) else f64(g["K"])
    plan = mb.build_varlen(g["topk"], len(g["counts"]))
    assert np.array_equal(plan.flat_queries, g["flat"])
    res = mb.moba_forward(Q, Kc, V, plan, cfg)
    assert_close(res.output, g["O"], f"{name} O")
    assert_close(res.logsumexp, g["LSE"], f"{name} LSE")
    dQ, dK, dV = mb.moba_backward(Q, Kc, V, res.output, dO, res.logsumexp, plan, cfg, schedule=schedule)
    assert_close(dQ, g["dQ"], f"{name} dQ")
    assert_close(dK, g["dK"], f"{name} dK")
    assert_close(dV, g["dV"], f"{name} dV")


@pytest.mark.parametrize("name", golden_names())
def test_end_to_end_vs_oracle_on_own_plan(name):
    """moba_attention end to end; the oracle re-runs the attention on the
    GPU's own plan (so routing near-ties cannot masquerade as errors)."""
    g = load(name)
    cfg = cfg_of(g)
    if int(g["width"]):
        pytest.skip("conv path covered by test_moba_attn_conv_autograd")
    Q, K, V = f64(g["Q"]), f64(g["K"]), f64(g["V"])
    res, plan = mb.moba_attention(Q, K, V, cfg)
    op = orc.OraclePlan(plan.topk_indices, plan.counts, plan.offsets, plan.flat_queries)
    O, L = orc.forward(Q, K, V, op, cfg.block_size_B)
    assert_close(res.output, O, "O")
    assert_close(res.logsumexp, L, "LSE")


def test_hand_tie_and_block0():
    for name in ("hand_tie", "hand_block0"):
        g = load(name)
        B, k = int(g["B"]), int(g["k"])
        d = g["Q"].shape[1]
        cfg = mb.MobaConfig(block_size_B=B, top_k=k, head_dim_d=d)
        idx = mb.select_topk(g["Q"], mb.compute_centroids(g["K"], B), cfg)
        assert np.array_equal(idx, g["topk"]), name


def test_plan_without_own_block():
    g = load("hand_no_own_block")
    cfg = mb.MobaConfig(block_size_B=int(g["B"]), top_k=1, head_dim_d=int(g["d"]))
    plan = mb.build_varlen(g["topk"], 4)
    Q, K, V, dO = (f64(g[x]) for x in ("Q", "K", "V", "dO"))
    res = mb.moba_forward(Q, K, V, plan, cfg)
    assert_close(res.output, g["O"], "O")
    assert_close(res.logsumexp, g["LSE"], "LSE")
    dQ, dK, dV = mb.moba_backward(Q, K, V, res.output, dO, res.logsumexp, plan, cfg)
    assert_close(dQ, g["dQ"], "dQ")
    B = int(g["B"])
    assert not dK[B:].any() and not dV[B:].any()      # tests/test_attention.py:246-247
    assert dK[:B].any() and dV[:B].any()


def test_invalid_plans_rejected():
    # tests/test_attention.py:179-193
    rng = np.random.default_rng(11)
    Q, K, V = (rng.standard_normal((64, 8)) for _ in range(3))
    cfg = mb.MobaConfig(block_size_B=16, top_k=2, head_dim_d=8)
    plan = mb.build_plan(Q, K, cfg)
    bad_idx = plan.topk_indices.copy()
    bad_idx[0, -1] = 3
    bad = mb.build_varlen(bad_idx, 4)
    with pytest.raises(mb.PlanValidationError):
        mb.moba_forward(Q, K, V, bad, cfg)
    broken = mb.build_plan(Q, K, cfg)
    broken.offsets = broken.offsets + 1
    with pytest.raises(mb.PlanValidationError):
        mb.moba_forward(Q, K, V, broken, cfg)
    with pytest.raises(mb.PlanValidationError):
        mb.build_varlen(np.array([[5]]), 3)
    with pytest.raises(mb.PlanValidationError):
        mb.build_varlen(np.array([[-2]]), 3)


def test_backward_zero_upstream_and_lse_checks():
    # tests/test_attention.py:205-210, :284-292
    rng = np.random.default_rng(12)
    Q, K, V = (rng.standard_normal((96, 8)) for _ in range(3))
    cfg = mb.MobaConfig(block_size_B=16, top_k=2, head_dim_d=8)
    res, plan = mb.moba_attention(Q, K, V, cfg)
    dQ, dK, dV = mb.moba_backward(Q, K, V, res.output, np.zeros_like(Q), res.logsumexp, plan, cfg)
    assert not dQ.any() and not dK.any() and not dV.any()
    with pytest.raises(mb.PlanValidationError):
        mb.moba_backward(Q, K, V, res.output, Q, res.logsumexp[:-1], plan, cfg)
    bad = res.logsumexp.copy()
    bad[0] = np.inf
    with pytest.raises(mb.PlanValidationError):
        mb.moba_backward(Q, K, V, res.output, Q, bad, plan, cfg)
    with pytest.raises(ValueError):
        mb.moba_backward(Q, K, V, res.output, Q, res.logsumexp, plan, cfg, schedule="bogus")


def test_deterministic_schedule_bitwise_repeatable():
    # tests/test_attention.py:276-282
    gen = torch.Generator(device="cuda").manual_seed(3)
    H, N, d = 4, 4096, 64
    q, k, v, do = (torch.randn(H, N, d, generator=gen, device="cuda").bfloat16() for _ in range(4))
    cfg = mb.MobaConfig(block_size_B=128, top_k=8, head_dim_d=d)
    res, plan = mb.moba_attention(q, k, v, cfg)
    a = mb.moba_backward(q, k, v, res.output, do, res.logsumexp, plan, cfg)
    b = mb.moba_backward(q, k, v, res.output, do, res.logsumexp, plan, cfg)
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    r2, _ = mb.moba_attention(q, k, v, cfg)
    assert torch.equal(res.output, r2.output) and torch.equal(res.logsumexp, r2.logsumexp)


def test_dense_limit_matches_dense_attention():
    # saturation: top_k >= n-1 -> plain causal attention (tests/test_attention.py:76-83)
    gen = torch.Generator(device="cuda").manual_seed(4)
    H, N, d = 2, 1024, 64
    q, k, v = (torch.randn(H, N, d, generator=gen, device="cuda").bfloat16() for _ in range(3))
    cfg = mb.MobaConfig(block_size_B=128, top_k=8, head_dim_d=d)
    res, plan = mb.moba_attention(q, k, v, cfg)
    ref = torch.nn.functional.scaled_dot_product_attention(q.float(), k.float(), v.float(), is_causal=True)
    assert_close(res.output.float().cpu().numpy(), ref.cpu().numpy(), "dense-limit O")


def test_c2_config_vs_oracle_sampled_heads():
    """BASELINE configs[1] (16 heads, N=8K, d=64, B=128, k=8): routing vs the
    f64 oracle on every head, fwd+bwd vs the oracle on the GPU plan (2 heads)."""
    gen = torch.Generator(device="cuda").manual_seed(0)
    H, N, d, B, k = 16, 8192, 64, 128, 8
    q, kk, v, do = (torch.randn(H, N, d, generator=gen, device="cuda").bfloat16() for _ in range(4))
    cfg = mb.MobaConfig(block_size_B=B, top_k=k, head_dim_d=d)
    res, plan = mb.moba_attention(q, kk, v, cfg)
    dq, dk, dv = mb.moba_backward(q, kk, v, res.output, do, res.logsumexp, plan, cfg, schedule="parallel")
    topk = plan.topk_indices
    Qn, Kn, Vn, dOn = (t.double().cpu().numpy() for t in (q, kk, v, do))
    total_diff = 0
    for h in range(H):
        c, _ = orc.centroids(Kn[h], B)
        ref_topk = orc.select_topk(Qn[h], c, B, k)
        bad, nd = unexcused_routing_rows(Qn[h], c, topk[h], ref_topk, B, k)
        assert not bad, (h, bad[:5])
        total_diff += nd
    for h in (0, H - 1):
        ph = plan.head(h)
        op = orc.OraclePlan(ph.topk_indices, ph.counts, ph.offsets, ph.flat_queries)
        O, L = orc.forward(Qn[h], Kn[h], Vn[h], op, B)
        assert_close(res.output[h].float().cpu().numpy(), O, f"O[{h}]")
        assert_close(res.logsumexp[h].cpu().numpy(), L, f"LSE[{h}]")
        rQ, rK, rV = orc.backward(Qn[h], Kn[h], Vn[h], res.output[h].double().cpu().numpy(), dOn[h],
                                  res.logsumexp[h].double().cpu().numpy(), op, B)
        assert_close(dq[h].float().cpu().numpy(), rQ, f"dQ[{h}]")
        assert_close(dk[h].float().cpu().numpy(), rK, f"dK[{h}]")
        assert_close(dv[h].float().cpu().numpy(), rV, f"dV[{h}]")


def test_moba_attn_conv_autograd():
    """Autograd path with the key conv (config 3 shape, scaled down) vs the oracle."""
    gen = torch.Generator(device="cuda").manual_seed(5)
    H, N, d, B, k, W = 2, 2048, 64, 64, 16, 3
    q, kk, v, do = (torch.randn(H, N, d, generator=gen, device="cuda").bfloat16() for _ in range(4))
    w = torch.tensor(orc.random_conv_weights(W, d, seed=7), dtype=torch.float32, device="cuda")
    q.requires_grad_(True), kk.requires_grad_(True), v.requires_grad_(True), w.requires_grad_(True)
    out, lse = mb.moba_attn(q, kk, v, B, k, conv_weight=w, return_lse=True)
    out.backward(do)
    Qn, Kn, Vn, dOn = (t.detach().double().cpu().numpy() for t in (q, kk, v, do))
    Wn = w.detach().double().cpu().numpy()
    for h in range(H):
        Kc = orc.key_conv_forward(Kn[h], Wn)
        c, _ = orc.centroids(Kc, B)
        plan_o = orc.build_plan(Qn[h], Kc, B, k)
        O, L = orc.forward(Qn[h], Kc, Vn[h], plan_o, B)
        # routing may differ only on ties; compare outputs where rows agree
        assert_close(out[h].detach().float().cpu().numpy(), O, f"conv O[{h}]")
        rQ, rKc, rV = orc.backward(Qn[h], Kc, Vn[h], O, dOn[h], L, plan_o, B)
        rK, _ = orc.key_conv_backward(Kn[h], Wn, rKc)
        assert_close(q.grad[h].float().cpu().numpy(), rQ, f"conv dQ[{h}]")
        assert_close(kk.grad[h].float().cpu().numpy(), rK, f"conv dK[{h}]")
        assert_close(v.grad[h].float().cpu().numpy(), rV, f"conv dV[{h}]")
    # dW summed over heads
    dW = 0
    for h in range(H):
        Kc = orc.key_conv_forward(Kn[h], Wn)
        plan_o = orc.build_plan(Qn[h], Kc, B, k)
        O, L = orc.forward(Qn[h], Kc, Vn[h], plan_o, B)
        _, rKc, _ = orc.backward(Qn[h], Kc, Vn[h], O, dOn[h], L, plan_o, B)
        dW = dW + orc.key_conv_backward(Kn[h], Wn, rKc)[1]
    # dW sums H x N terms g * K, so |dW| grows with H*N while every term
    # carries the bf16-level error of dK' from the attention backward: the
    # 2e-2 contract is applied relative to the largest entry
    assert_close(w.grad.cpu().numpy(), dW, "conv dW", max_abs=2e-2 * max(1.0, float(np.abs(dW).max())))


def test_key_conv_backward_vs_reference():
    for name in ("conv3_n512_b64", "conv5_n300_b32"):
        g = load(name)
        dK, dW = mb.key_conv_backward(f64(g["K"]), mb.ConvKernel(g["W"]), f64(g["dO"]))
        # dK comes back from its bf16 kernel copy: elementwise 2^-8 |dK|
        # (round-to-nearest bf16 is within 2^-9) + 1e-5 for the fp32 math;
        # dW is fp32: the 2e-2 contract relative to its largest entry (a sum
        # over N tokens)
        err = np.abs(np.asarray(dK, np.float64) - g["conv_dK"])
        assert np.all(err <= 2.0 ** -8 * np.abs(g["conv_dK"]) + 1e-5), name
        assert_close(dW, g["conv_dW"], f"{name} conv dW", max_abs=2e-2 * max(1.0, float(np.abs(g["conv_dW"]).max())))


@pytest.mark.slow
def test_full_size_64k_properties():
    """Metric-size plan (N=64K, B=128, k=8): size-independent properties —
    conservation, prefix sums, ascending slices, causality, own block present,
    and routing vs the f64 oracle on a sample of query rows."""
    gen = torch.Generator(device="cuda").manual_seed(0)
    H, N, d, B, k = 2, 65536, 64, 128, 8
    q, kk, v = (torch.randn(H, N, d, generator=gen, device="cuda").bfloat16() for _ in range(3))
    cfg = mb.MobaConfig(block_size_B=B, top_k=k, head_dim_d=d)
    res, plan = mb.moba_attention(q, kk, v, cfg)
    assert bool(torch.isfinite(res.output.float()).all()) and bool(torch.isfinite(res.logsumexp).all())
    E = orc.plan_entries(N, B, k)
    counts = plan.counts_d.long()
    assert int(counts.sum()) == H * E
    topk = plan.topk.long()
    i = torch.arange(N, device="cuda").view(1, N, 1)
    assert bool(((topk <= i // B) | (topk < 0)).all())
    assert bool((topk == (i // B)).any(dim=2).all())
    mb.validate_plan(plan, N, cfg)
    Qn, Kn = q.double().cpu().numpy(), kk.double().cpu().numpy()
    rows = np.random.default_rng(0).choice(N, 2048, replace=False)
    rows.sort()
    for h in range(H):
        c, _ = orc.centroids(Kn[h], B)
        got = plan.topk_indices[h]
        ref = got.copy()
        ref[rows] = _select_rows(Qn[h], c, B, k, rows)   # only sampled rows can differ
        bad, _ = unexcused_routing_rows(Qn[h], c, got, ref, B, k)
        assert not bad, bad[:5]


def _select_rows(Q, c, B, k, rows):
    out = np.full((len(rows), k + 1), -1, np.int32)
    own = rows // B
    sel = orc._topk_rows(Q[rows] @ c.T, own, k)
    sel[np.arange(len(rows)), own] = True
    for r in range(len(rows)):
        ids = np.nonzero(sel[r])[0]
        out[r, : len(ids)] = ids
    return out


@pytest.mark.parametrize("name", golden_names())
def test_routing_tensor_core_mode_vs_reference(name):
    """Perf routing mode (bf16x3 centroid split on tcgen05): same selections as
    the reference up to score near-ties (the 1e-6 contract on the f64 score
    gap)."""
    g = load(name)
    if int(g["d"]) > 128:
        pytest.skip("d > 128")
    B, k, width = int(g["B"]), int(g["k"]), int(g["width"])
    from paper_2511_11571_b200 import _device
    dp = _device.padded_dim(int(g["d"]))
    pad = lambda t: torch.nn.functional.pad(t, (0, dp - t.shape[-1])).contiguous()
    qt = pad(torch.tensor(g["Q"]).cuda().bfloat16()[None])
    kt = pad(torch.tensor(g["K"]).cuda().bfloat16()[None])
    w = pad(torch.tensor(g["W"], dtype=torch.float32).cuda()) if width else None
    cent, _ = _device.centroids(kt, B, w)
    plan = _device.route(qt, cent, B, k, mode=1)
    bad, ndiff = unexcused_routing_rows(f64(g["Q"]), g["centroids"], plan.topk_indices, g["topk"], B, k)
    assert not bad, f"{len(bad)} rows differ beyond ties (of {ndiff}): {bad[:10]}"
    orc.validate_plan(orc.OraclePlan(plan.topk_indices, plan.counts, plan.offsets, plan.flat_queries),
                      int(g["N"]), B)


def test_routing_tensor_core_mode_c2_scale():
    gen = torch.Generator(device="cuda").manual_seed(11)
    H, N, d, B, k = 4, 8192, 64, 128, 8
    q, kk = (torch.randn(H, N, d, generator=gen, device="cuda").bfloat16() for _ in range(2))
    cfg = mb.MobaConfig(block_size_B=B, top_k=k, head_dim_d=d)
    p_tc = mb.build_plan(q, kk, cfg, mode="tc")
    p_fp = mb.build_plan(q, kk, cfg, mode="fp32")
    Qn, Kn = q.double().cpu().numpy(), kk.double().cpu().numpy()
    for h in range(H):
        c, _ = orc.centroids(Kn[h], B)
        bad, nd = unexcused_routing_rows(Qn[h], c, p_tc.topk_indices[h], p_fp.topk_indices[h], B, k)
        assert not bad, (h, bad[:5], nd)


@pytest.mark.parametrize("graphs", [False, True])
@pytest.mark.parametrize("n_chunks", [1, 3, None])
def test_host_pipeline_matches_device_path(n_chunks, graphs):
    """moba_fwd_bwd_host (pinned host buffers, chunked over heads, copies on
    their own streams) returns bitwise the device path's results."""
    gen = torch.Generator(device="cuda").manual_seed(11)
    H, N, d, B, k = 5, 2048, 64, 128, 8
    q, kk, v, do = (torch.randn(H, N, d, generator=gen, device="cuda").bfloat16() for _ in range(4))
    qg, kg, vg = (t.clone().requires_grad_(True) for t in (q, kk, v))
    out, lse = mb.moba_attn(qg, kg, vg, B, k, mode="tc", deterministic=True, return_lse=True)
    out.backward(do)
    host = [t.cpu().pin_memory() for t in (q, kk, v, do)]
    for _ in range(2):   # the second call reuses the captured chunk graphs
        o_h, lse_h, dq_h, dk_h, dv_h = mb.moba_fwd_bwd_host(*host, B, k, n_chunks=n_chunks, mode="tc",
                                                            deterministic=True, graphs=graphs)
    for got, ref, nm in ((o_h, out, "O"), (lse_h, lse, "LSE"), (dq_h, qg.grad, "dQ"), (dk_h, kg.grad, "dK"),
                         (dv_h, vg.grad, "dV")):
        assert not got.is_cuda
        assert torch.equal(got, ref.detach().cpu()), nm


@pytest.mark.parametrize("conv,d,B", [(False, 64, 128), (True, 64, 128), (False, 128, 128), (False, 64, 256)])
def test_graphed_step_matches_eager(conv, d, B):
    """MobaGraphedStep (the whole fwd+bwd captured once, replayed) gives
    bitwise the eager results, also after the inputs change (a new plan).
    d = 128 runs the other backward kernel (its debug-trace pointer once went
    through a host-memory copy that a captured graph replayed from a stale
    stack address)."""
    gen = torch.Generator(device="cuda").manual_seed(5)
    H, N, k = 3, 1536, 4
    w = (torch.rand(3, d, generator=gen, device="cuda") - 0.5) if conv else None
    gs = mb.MobaGraphedStep((H, N, d), B, k, mode="tc", deterministic=True, conv_weight=w)
    for trial in range(2):
        q, kk, v, do = (torch.randn(H, N, d, generator=gen, device="cuda").bfloat16() for _ in range(4))
        out, dq, dk, dv = gs.step(q, kk, v, do)
        qg, kg, vg = (t.clone().requires_grad_(True) for t in (q, kk, v))
        ref = mb.moba_attn(qg, kg, vg, B, k, mode="tc", deterministic=True, conv_weight=w)
        ref.backward(do)
        for got, exp, nm in ((out, ref, "O"), (dq, qg.grad, "dQ"), (dk, kg.grad, "dK"), (dv, vg.grad, "dV")):
            assert torch.equal(got, exp), (trial, nm)


@pytest.mark.parametrize("hq,hkv,d,B", [(8, 2, 64, 128), (4, 1, 64, 64), (4, 2, 128, 128)])
def test_gqa_matches_expanded_heads(hq, hkv, d, B):
    """GQA/MQA: K/V heads shared by hq/hkv query heads give
    the same O/LSE/dQ as running MHA on repeated K/V heads, and dK/dV equal
    the per-group sums of the repeated heads' gradients."""
    gen = torch.Generator(device="cuda").manual_seed(21)
    N, k = 1280, 4
    G = hq // hkv
    q, do = (torch.randn(2, hq, N, d, generator=gen, device="cuda").bfloat16() for _ in range(2))
    kk, v = (torch.randn(2, hkv, N, d, generator=gen, device="cuda").bfloat16() for _ in range(2))
    qg, kg, vg = (t.clone().requires_grad_(True) for t in (q, kk, v))
    out, lse = mb.moba_attn(qg, kg, vg, B, k, mode="fp32", deterministic=True, return_lse=True)
    out.backward(do)
    qe = q.clone().requires_grad_(True)
    ke = kk.repeat_interleave(G, dim=1).requires_grad_(True)
    ve = v.repeat_interleave(G, dim=1).requires_grad_(True)
    oe, lse_e = mb.moba_attn(qe, ke, ve, B, k, mode="fp32", deterministic=True, return_lse=True)
    oe.backward(do)
    assert torch.equal(out, oe) and torch.equal(lse, lse_e)
    assert torch.equal(qg.grad, qe.grad)
    for got, exp, nm in ((kg.grad, ke.grad, "dK"), (vg.grad, ve.grad, "dV")):
        ref = exp.float().view(2, hkv, G, N, d).sum(2).bfloat16().float()   # one bf16 rounding of the sum
        assert got.shape == kk.shape
        assert_close(got.float().cpu().numpy(), ref.cpu().numpy(), nm, max_abs=1e-2, rel=1e-3)


def test_gqa_vs_oracle():
    """GQA against the CPU oracle: each query head attends with its K/V
    head; dK/dV of a K/V head = sum of the oracle's per-query-head dK/dV."""
    gen = torch.Generator(device="cuda").manual_seed(22)
    hq, hkv, N, d, B, k = 4, 2, 700, 64, 64, 3
    q, do = (torch.randn(hq, N, d, generator=gen, device="cuda").bfloat16() for _ in range(2))
    kk, v = (torch.randn(hkv, N, d, generator=gen, device="cuda").bfloat16() for _ in range(2))
    qg, kg, vg = (t.clone().requires_grad_(True) for t in (q, kk, v))
    out = mb.moba_attn(qg, kg, vg, B, k, mode="fp32", deterministic=True)
    out.backward(do)
    Qn, Kn, Vn, dOn = (t.double().cpu().numpy() for t in (q, kk, v, do))
    dK = np.zeros_like(Kn)
    dV = np.zeros_like(Vn)
    for h in range(hq):
        hk = h // (hq // hkv)
        plan = orc.build_plan(Qn[h], Kn[hk], B, k)
        O, L = orc.forward(Qn[h], Kn[hk], Vn[hk], plan, B)
        dq, dk, dv = orc.backward(Qn[h], Kn[hk], Vn[hk], O, dOn[h], L, plan, B)
        assert_close(out[h].detach().double().cpu().numpy(), O, f"O[{h}]")
        assert_close(qg.grad[h].double().cpu().numpy(), dq, f"dQ[{h}]")
        dK[hk] += dk
        dV[hk] += dv
    assert_close(kg.grad.double().cpu().numpy(), dK, "dK")
    assert_close(vg.grad.double().cpu().numpy(), dV, "dV")


def test_hybrid_lm_train_step():
    """C5 layer stack at toy size: SWA+RoPE / MoBA(+kconv3)
    alternating layers train end to end through the MoBA kernels (loss falls
    on a repeated batch; every MoBA-layer parameter gets a finite gradient)."""
    pytest.importorskip("flash_attn")
    from paper_2511_11571_b200.lm import MobaLM, MobaLMConfig, train_step
    torch.manual_seed(0)
    cfg = MobaLMConfig(vocab=512, hidden=256, heads=4, head_dim=64, intermediate=512, layers=4, block_size=128,
                       top_k=4, conv_width=3)
    model = MobaLM(cfg).cuda().to(torch.bfloat16)
    opt = torch.optim.AdamW(model.parameters(), lr=3e-3)
    tokens = torch.randint(0, cfg.vocab, (2, 1024), device="cuda")
    losses = [float(train_step(model, opt, tokens)) for _ in range(12)]
    assert all(np.isfinite(losses)), losses
    assert min(losses[-3:]) < losses[0] - 0.2, losses
    model.zero_grad()
    model.loss(tokens).backward()
    blk = model.blocks[1]            # layer 2: MoBA with key conv
    assert blk.attn.moba and blk.attn.conv is not None
    for name, p in blk.named_parameters():
        assert p.grad is not None and bool(torch.isfinite(p.grad).all()) and float(p.grad.abs().sum()) > 0, name


def test_cli_attend_tns1_vs_oracle(tmp_path):
    """`cli attend` on TNS1 files: output, LSE and the
    emitted plan match the oracle (single head, key conv on)."""
    import json as _json
    from paper_2511_11571_b200 import cli
    from paper_2511_11571_b200.tensorio import Tensor, tensor_read, tensor_write
    rng = np.random.default_rng(3)
    N, d, B, k, W = 640, 64, 64, 3, 3
    Q, K, V = (bf16_round(rng.standard_normal((N, d))) for _ in range(3))
    w = rng.uniform(-0.5, 0.5, size=(W, d))
    for name, arr in (("q", Q), ("k", K), ("v", V), ("w", w)):
        tensor_write(Tensor(arr), tmp_path / f"{name}.tns")
    rc = cli.main(["attend", "--q", str(tmp_path / "q.tns"), "--k", str(tmp_path / "k.tns"), "--v",
                   str(tmp_path / "v.tns"), "--out", str(tmp_path / "o.tns"), "--block", str(B), "--topk", str(k),
                   "--conv", str(W), "--kernel", str(tmp_path / "w.tns"), "--emit-plan", str(tmp_path / "p.json"),
                   "--emit-lse", str(tmp_path / "l.tns")])
    assert rc == 0
    Kc = orc.key_conv_forward(K, w)
    plan = orc.build_plan(Q, Kc, B, k)
    O, L = orc.forward(Q, Kc, V, plan, B)
    assert_close(tensor_read(tmp_path / "o.tns").array, O, "O")
    assert_close(tensor_read(tmp_path / "l.tns").array, L, "LSE")
    p = _json.load(open(tmp_path / "p.json"))
    assert p["counts"] == plan.counts.tolist()
    assert p["offsets"] == plan.offsets.tolist()
    assert p["flat_queries"] == plan.flat_queries.tolist()


@pytest.mark.parametrize("N,B,k,d", [(1536, 256, 4, 64), (2048, 512, 2, 64), (1000, 200, 3, 64), (1024, 256, 2, 128)])
def test_large_blocks_vs_oracle(N, B, k, d):
    """Key blocks longer than 128 keys (the paper's MoBA-256 / MoBA-512,
    PAPER.md:317-320): the forward runs them as 128-key slabs with one
    partial each; fwd + bwd against the oracle."""
    gen = torch.Generator(device="cuda").manual_seed(B + k)
    H = 2
    q, kk, v, do = (torch.randn(H, N, d, generator=gen, device="cuda").bfloat16() for _ in range(4))
    qg, kg, vg = (t.clone().requires_grad_(True) for t in (q, kk, v))
    out, lse = mb.moba_attn(qg, kg, vg, B, k, mode="fp32", deterministic=True, return_lse=True)
    out.backward(do)
    Qn, Kn, Vn, dOn = (t.double().cpu().numpy() for t in (q, kk, v, do))
    for h in range(H):
        plan = orc.build_plan(Qn[h], Kn[h], B, k)
        O, L = orc.forward(Qn[h], Kn[h], Vn[h], plan, B)
        dQ, dK, dV = orc.backward(Qn[h], Kn[h], Vn[h], O, dOn[h], L, plan, B)
        for got, ref, nm in ((out[h], O, "O"), (lse[h], L, "LSE"), (qg.grad[h], dQ, "dQ"), (kg.grad[h], dK, "dK"),
                             (vg.grad[h], dV, "dV")):
            assert_close(got.detach().double().cpu().numpy(), ref, f"{nm}[{h}] B={B}")


def _sweep_cases(n=16, seed=2024):
    rng = np.random.default_rng(seed)
    cases = []
    for _ in range(n):
        B = int(rng.choice([16, 32, 64, 96, 128, 192, 256, 512]))
        N = int(rng.integers(B // 2 + 1, 6 * B + 1))
        k = int(rng.integers(1, 9))
        d = int(rng.choice([16, 32, 64, 100, 128]))
        hkv = int(rng.choice([1, 2]))
        G = int(rng.choice([1, 2, 3]))
        conv = int(rng.choice([0, 0, 3, 5]))
        cases.append((N, B, k, d, hkv, G, conv, bool(rng.integers(0, 2))))
    return cases


@pytest.mark.parametrize("N,B,k,d,hkv,G,conv,det", _sweep_cases())
def test_randomized_sweep_vs_oracle(N, B, k, d, hkv, G, conv, det):
    """Seeded random sweep over shapes (ragged N, B up to 512, d padded to
    64/128, GQA groups, key conv, both dQ schedules): fp32 routing matches the
    oracle's plan up to documented ties; O/LSE/dQ/dK/dV within tolerance."""
    gen = torch.Generator(device="cuda").manual_seed(N * 7 + B)
    hq = hkv * G
    q, do = (torch.randn(hq, N, d, generator=gen, device="cuda").bfloat16() for _ in range(2))
    kk, v = (torch.randn(hkv, N, d, generator=gen, device="cuda").bfloat16() for _ in range(2))
    w = (torch.rand(conv, d, generator=gen, device="cuda") - 0.5) if conv else None
    qg, kg, vg = (t.clone().requires_grad_(True) for t in (q, kk, v))
    out, lse = mb.moba_attn(qg, kg, vg, B, k, conv_weight=w, mode="fp32", deterministic=det, return_lse=True)
    out.backward(do)
    Qn, Kn, Vn, dOn = (t.double().cpu().numpy() for t in (q, kk, v, do))
    Wn = w.double().cpu().numpy() if conv else None
    dK = np.zeros_like(Kn)
    dV = np.zeros_like(Vn)
    for h in range(hq):
        hk = h // G
        Kc = orc.key_conv_forward(Kn[hk], Wn) if conv else Kn[hk]
        plan = orc.build_plan(Qn[h], Kc, B, k)
        O, L = orc.forward(Qn[h], Kc, Vn[hk], plan, B)
        dq, dkc, dv = orc.backward(Qn[h], Kc, Vn[hk], O, dOn[h], L, plan, B)
        dk = orc.key_conv_backward(Kn[hk], Wn, dkc)[0] if conv else dkc
        tag = f"h{h} N{N} B{B} k{k} d{d} G{G} conv{conv}"
        assert_close(out[h].detach().double().cpu().numpy(), O, "O " + tag)
        assert_close(lse[h].detach().double().cpu().numpy(), L, "LSE " + tag)
        assert_close(qg.grad[h].double().cpu().numpy(), dq, "dQ " + tag)
        dK[hk] += dk
        dV[hk] += dv
    # dK / dV of a K/V head sum G query heads' gradients (and are rounded to
    # bf16 once at the larger magnitude): the absolute tolerance scales with G
    assert_close(kg.grad.double().cpu().numpy(), dK, "dK", max_abs=2e-2 * G)
    assert_close(vg.grad.double().cpu().numpy(), dV, "dV", max_abs=2e-2 * G)


def test_plan_with_disagreeing_layouts_rejected():
    """A plan whose topk_indices name a (query, block) pair that flat_queries
    does not list — with every count, offset and total still consistent —
    is a PlanValidationError (src/core.py:254-296 checks both layouts)."""
    rng = np.random.default_rng(13)
    N, d, B, k = 512, 16, 32, 3
    Q, K, V = (rng.standard_normal((N, d)) for _ in range(3))
    cfg = mb.MobaConfig(block_size_B=B, top_k=k, head_dim_d=d)
    plan = mb.build_plan(Q, K, cfg)
    idx = plan.topk_indices.copy()
    i = N - 1
    row = idx[i]
    unused = [j for j in range(i // B) if j not in set(row.tolist())]
    # move one routed block of query i to a block it did not pick: the row
    # stays unique and causal, the totals are unchanged, flat still lists
    # the old block
    row[0] = unused[0]
    idx[i] = np.sort(row)
    plan.topk_indices = idx
    with pytest.raises(mb.PlanValidationError):
        mb.validate_plan(plan, N, cfg)
    with pytest.raises(mb.PlanValidationError):
        mb.moba_forward(Q, K, V, plan, cfg)


def test_generic_f64_inputs_route_unrounded():
    """numpy f64 inputs that are NOT bf16-representable: centroids and fp32
    routing use the unrounded values, so the plan matches the f64 oracle up
    to 1e-6 ties (rounding Q / K to bf16 first would move selections by
    ~1e-2 score gaps); O / LSE / dQ / dK / dV stay within the 2e-2 contract."""
    rng = np.random.default_rng(14)
    N, d, B, k = 4096, 64, 64, 6
    Q, K, V, dO = (rng.standard_normal((N, d)) for _ in range(4))
    cfg = mb.MobaConfig(block_size_B=B, top_k=k, head_dim_d=d)
    res, plan = mb.moba_attention(Q, K, V, cfg)
    c, _ = orc.centroids(K, B)
    ref = orc.select_topk(Q, c, B, k)
    bad, nd = unexcused_routing_rows(Q, c, plan.topk_indices, ref, B, k)
    assert not bad, (len(bad), nd, bad[:5])
    cents = mb.compute_centroids(K, B)
    np.testing.assert_allclose(cents.centroids, c, rtol=1e-6, atol=1e-7)
    op = orc.OraclePlan(plan.topk_indices, plan.counts, plan.offsets, plan.flat_queries)
    O, L = orc.forward(Q, K, V, op, B)
    assert_close(res.output, O, "O")
    assert_close(res.logsumexp, L, "LSE")
    dQ, dK, dV = mb.moba_backward(Q, K, V, res.output, dO, res.logsumexp, plan, cfg)
    rQ, rK, rV = orc.backward(Q, K, V, O, dO, L, op, B)
    assert_close(dQ, rQ, "dQ")
    assert_close(dK, rK, "dK")
    assert_close(dV, rV, "dV")


def test_head_view_of_stale_plan_rebuilds_row_pos():
    """RoutingPlan.head() of a plan whose fields were reassigned does not
    inherit the stale (query, slot) -> flat position map."""
    gen = torch.Generator(device="cuda").manual_seed(15)
    H, N, d, B, k = 2, 1024, 64, 128, 3
    q, kk, v = (torch.randn(H, N, d, generator=gen, device="cuda").bfloat16() for _ in range(3))
    cfg = mb.MobaConfig(block_size_B=B, top_k=k, head_dim_d=d)
    plan = mb.build_plan(q, kk, cfg)
    other = mb.build_plan(torch.flip(q, dims=[0]), kk, cfg)
    plan.topk_indices = other.topk_indices
    plan.counts, plan.offsets, plan.flat_queries = other.counts, other.offsets, other.flat_queries
    h1 = plan.head(1)
    assert h1.row_pos is None
    res = mb.moba_forward(q[1:], kk[1:], v[1:], h1, cfg)
    ref = mb.moba_forward(q[1:], kk[1:], v[1:], other.head(1), cfg)
    assert torch.equal(res.output, ref.output)


def test_moba_forward_backward_accept_reference_plan():
    """A plan object shaped like the reference's RoutingPlan dataclass
    (src/core.py:229-251: numpy topk_indices / counts / offsets /
    flat_queries for one head) drives moba_forward / moba_backward exactly
    like this package's plan; a malformed one raises PlanValidationError."""
    from types import SimpleNamespace
    g = load("ragged_n500_b64")
    cfg = mb.MobaConfig(block_size_B=int(g["B"]), top_k=int(g["k"]), head_dim_d=g["Q"].shape[1])
    ref_plan = SimpleNamespace(topk_indices=g["topk"], counts=g["counts"], offsets=g["offsets"], flat_queries=g["flat"])
    Q, K, V = f64(g["Q"]), f64(g["K"]), f64(g["V"])
    res = mb.moba_forward(Q, K, V, ref_plan, cfg)
    assert_close(res.output, g["O"], "O (reference-shaped plan)")
    assert_close(res.logsumexp, g["LSE"], "LSE (reference-shaped plan)")
    dQ, dK, dV = mb.moba_backward(Q, K, V, res.output, f64(g["dO"]), res.logsumexp, ref_plan, cfg)
    assert_close(dQ, g["dQ"], "dQ (reference-shaped plan)")
    assert_close(dK, g["dK"], "dK (reference-shaped plan)")
    assert_close(dV, g["dV"], "dV (reference-shaped plan)")
    bad = SimpleNamespace(topk_indices=g["topk"], counts=g["counts"], offsets=g["offsets"], flat_queries=g["flat"][:-1])
    with pytest.raises(mb.PlanValidationError):
        mb.moba_forward(Q, K, V, bad, cfg)
