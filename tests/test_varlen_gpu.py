"""build_varlen on the GPU (moba_varlen: count / scan / wide-chunk scatter,
router.cu) against the oracle's stable counting sort (oracle/moba_oracle.py
build_varlen, src/router.py:123-154): counts, offsets, flat_queries and the
row_pos inverse map must be bit-exact.

The index rows are drawn at random — not only causal router output: any
block in [0, n) per slot, distinct within a row, -1 padding anywhere — so the
chunk geometry (several chunks per head, 2..16 walking warps, chunk sizes
grown from 128 to 2048 queries) is exercised on rows the router never emits.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import moba_oracle as orc  # noqa: E402
from paper_2511_11571_b200 import _device  # noqa: E402


def _rows(rng, N, n, width, causal, B):
    out = np.full((N, width), -1, dtype=np.int32)
    for i in range(N):
        hi = i // B + 1 if causal else n
        m = int(rng.integers(0, min(width, hi) + 1))
        sel = np.sort(rng.choice(hi, size=m, replace=False)) if m else np.zeros(0, dtype=np.int64)
        slots = np.sort(rng.choice(width, size=m, replace=False)) if not causal else np.arange(m)
        out[i, slots] = sel
    return out


def _check(topk_h, plan, h, n):
    ref = orc.build_varlen(topk_h, n)
    tot = int(ref.counts.sum())
    assert np.array_equal(plan.counts_d[h].cpu().numpy(), ref.counts)
    assert np.array_equal(plan.offsets_d[h].cpu().numpy(), ref.offsets)
    assert np.array_equal(plan.flat_d[h, :tot].cpu().numpy(), ref.flat_queries)
    # row_pos: flat position of each (query, slot) entry, -1 for padding
    rp = plan.row_pos[h].cpu().numpy()
    valid = topk_h >= 0
    assert np.all(rp[~valid] == -1)
    q = np.nonzero(valid)[0]
    assert np.array_equal(ref.flat_queries[rp[valid]], q.astype(np.int32))
    assert np.array_equal(np.searchsorted(ref.offsets, rp[valid], side="right") - 1, topk_h[valid])


@pytest.mark.parametrize("H,N,B,width,causal", [
    (3, 5000, 125, 9, False),      # non-causal rows, one head's chunks of 128 queries
    (2, 20000, 64, 17, False),     # wide rows (top-16)
    (1, 3001, 16, 32, False),      # widest rows, n = 188
    (4, 40000, 128, 9, True),      # causal, several 512-query chunks per head
    (1, 70000, 32, 5, True),       # n = 2188
])
def test_varlen_matches_oracle(H, N, B, width, causal):
    rng = np.random.default_rng(N + width)
    n = -(-N // B)
    topk = np.stack([_rows(rng, N, n, width, causal, B) for _ in range(H)])
    plan = _device.varlen(torch.from_numpy(topk).cuda(), B)
    torch.cuda.synchronize()
    for h in range(H):
        _check(topk[h], plan, h, n)


def _causal_topk(H, N, B, k, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    own = torch.arange(N, device="cuda") // B
    n = int(own.max().item()) + 1
    # k distinct past blocks per row (fewer near the start), sorted, then own;
    # scores drawn per (row, block) in row slabs to bound memory
    rows = []
    for h in range(H):
        sel_h = []
        for r0 in range(0, N, 8192):
            o = own[r0:r0 + 8192]
            r = torch.rand(o.numel(), n, device="cuda", generator=g)
            r = torch.where(torch.arange(n, device="cuda")[None, :] < o[:, None], r, -1.0)
            top = torch.topk(r, min(k, n), dim=1)
            sel = torch.where(top.values >= 0, top.indices, torch.full_like(top.indices, 1 << 30))
            sel = torch.sort(sel, dim=1).values
            sel_h.append(torch.where(sel == (1 << 30), torch.full_like(sel, -1), sel))
        rows.append(torch.cat(sel_h))
    sel = torch.stack(rows)
    return torch.cat([sel, own[None, :, None].expand(H, N, 1)], dim=2).int().contiguous()


def _check_torch_sort(topk, plan, B):
    H, N, W = topk.shape
    for h in range(H):
        t = topk[h].reshape(-1).long()
        q = torch.arange(N, device="cuda").repeat_interleave(W)
        ok = t >= 0
        key = torch.where(ok, t * N + q, torch.full_like(t, 1 << 62))
        srt, perm = torch.sort(key, stable=True)
        nv = int(ok.sum())
        assert torch.equal(plan.flat_d[h, :nv], (srt[:nv] % N).int())
        rp = torch.full_like(t, -1)
        rp[perm[:nv]] = torch.arange(nv, device="cuda")
        assert torch.equal(plan.row_pos[h].reshape(-1), rp.int())
        assert torch.equal(plan.counts_d[h], torch.bincount(t[ok], minlength=-(-N // B)).int())


@pytest.mark.parametrize("H,N,B,k", [
    (8, 65536, 128, 8),     # the metric shape's plan geometry: n = 512, 512-query chunks, 16 walking warps
    (1, 524288, 32, 16),    # n = 16384, 17-wide rows: the cursor words do not fit, one-warp fallback
])
def test_varlen_causal_torch_sort(H, N, B, k):
    """Causal top-k rows (the router's row format) against a torch.sort of
    the (block, query) pairs on the device."""
    topk = _causal_topk(H, N, B, k, seed=N + k)
    plan = _device.varlen(topk, B)
    _check_torch_sort(topk, plan, B)
