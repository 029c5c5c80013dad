"""The tensor-core router (tcgen05 scores from a two-term bf16 split of the
centroids, route_tc.cu) is certified against the fp32 router: its guard
(score gap vs a per-row error bound, in-kernel exact rescoring of the k + 2
best candidates, exact fp32 re-routing of undecided tiles) makes its plan
BITWISE the fp32 router's plan — and the fp32 router is the one held to
the reference (ties within 1e-6, tests/test_gpu_parity.py). Checked over
shapes, GQA, key conv, exact ties (repeated key blocks) and badly scaled
inputs."""
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2511_11571_b200 import _device, _lib  # noqa: E402


def _plans(q, k, B, topk, w=None):
    cent, _ = _device.centroids(k, B, w)
    return (_device.route(q, cent, B, topk, _lib.MOBA_ROUTE_TC), _device.route(q, cent, B, topk, _lib.MOBA_ROUTE_FP32))


def _same(a, b):
    assert torch.equal(a.topk, b.topk), int((a.topk != b.topk).any(dim=2).sum())
    assert torch.equal(a.counts_d, b.counts_d) and torch.equal(a.offsets_d, b.offsets_d)
    assert torch.equal(a.row_pos, b.row_pos)
    tot = a.counts_d.long().sum(dim=1)
    for h in range(a.topk.shape[0]):        # flat_d beyond a head's entries is unused capacity
        assert torch.equal(a.flat_d[h, : int(tot[h])], b.flat_d[h, : int(tot[h])])


@pytest.mark.parametrize("H,N,d,B,k", [(4, 8192, 64, 128, 8), (2, 65536, 64, 128, 8), (2, 16384, 128, 128, 8),
                                       (2, 32768, 64, 64, 16), (3, 1000, 64, 32, 3), (2, 4096, 128, 256, 4),
                                       (2, 3000, 64, 16, 1), (1, 20000, 64, 32, 31), (2, 9000, 128, 64, 2),
                                       (1, 131072, 64, 16, 8), (2, 300, 64, 128, 8), (5, 1500, 128, 32, 8),
                                       (1, 262144, 64, 128, 8), (1, 300000, 64, 64, 16)])
def test_tc_plan_equals_fp32_plan(H, N, d, B, k):
    gen = torch.Generator(device="cuda").manual_seed(N + k)
    q, kk = (torch.randn(H, N, d, generator=gen, device="cuda").bfloat16() for _ in range(2))
    _same(*_plans(q, kk, B, k))


def test_tc_plan_exact_ties_and_gqa():
    """Repeated key blocks give exactly equal centroids (exact score ties:
    the lower block index must win, src/router.py:95-98); GQA shares them."""
    gen = torch.Generator(device="cuda").manual_seed(3)
    Hq, Hk, N, d, B, k = 4, 2, 16384, 64, 128, 8
    base = torch.randn(Hk, 7 * B, d, generator=gen, device="cuda").bfloat16()
    reps = -(-N // (7 * B))
    kk = base.repeat(1, reps, 1)[:, :N].contiguous()
    q = torch.randn(Hq, N, d, generator=gen, device="cuda").bfloat16()
    _same(*_plans(q, kk, B, k))


@pytest.mark.parametrize("scale_q,scale_k", [(64.0, 1.0), (1.0, 1e-3), (1e-2, 30.0)])
def test_tc_plan_badly_scaled(scale_q, scale_k):
    gen = torch.Generator(device="cuda").manual_seed(4)
    q = (torch.randn(2, 8192, 64, generator=gen, device="cuda") * scale_q).bfloat16()
    kk = (torch.randn(2, 8192, 64, generator=gen, device="cuda") * scale_k).bfloat16()
    _same(*_plans(q, kk, 128, 8))


def test_tc_plan_with_key_conv():
    gen = torch.Generator(device="cuda").manual_seed(5)
    q, kk = (torch.randn(2, 32768, 64, generator=gen, device="cuda").bfloat16() for _ in range(2))
    w = (torch.rand(3, 64, generator=gen, device="cuda") - 0.5).contiguous()
    _same(*_plans(q, kk, 64, 16, w))


@pytest.mark.parametrize("kind", ["zeros", "constant_keys", "padded_tail"])
def test_tc_plan_degenerate_inputs(kind):
    """All-tie inputs (zero / constant keys, a zero-padded tail as in padded
    training batches): every affected row is undecidable for the
    tensor-core scores, so its tile is routed again by the exact fp32 router
    (tile-list mode) — the plan is still bitwise the fp32 router's, and the
    pass stays far cheaper than a per-row reselection (timed below)."""
    gen = torch.Generator(device="cuda").manual_seed(6)
    H, N, d, B, k = 8, 65536, 64, 128, 8
    q = torch.randn(H, N, d, generator=gen, device="cuda").bfloat16()
    kk = torch.randn(H, N, d, generator=gen, device="cuda").bfloat16()
    if kind == "zeros":
        q.zero_()
        kk.zero_()
    elif kind == "constant_keys":
        kk[:] = kk[:, :1, :]
    else:
        q[:, N // 2:] = 0
        kk[:, N // 2:] = 0
    tc, fp = _plans(q, kk, B, k)
    _same(tc, fp)
    cent, _ = _device.centroids(kk, B)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _device.route(q, cent, B, k, _lib.MOBA_ROUTE_TC)
    b.record()
    torch.cuda.synchronize()
    assert a.elapsed_time(b) < 50.0, f"degenerate tc routing took {a.elapsed_time(b):.1f} ms"
