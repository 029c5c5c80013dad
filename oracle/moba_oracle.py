"""CPU oracle for the MoBA attention hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package's algorithm
(`/root/reference/pkg/src/moba`, cited below as `src/<file>:<line>`). It is
the checker the CUDA path is compared against. Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl
reference` leg may import it; the product package `paper_2511_11571_b200`
never does (its ops raise if the CUDA library is missing).

Parity pin: every function here is checked bit-for-bit (integer outputs) or
to <=1e-12 (f64 outputs) against fixtures produced by the reference itself
(`tests/golden/make_golden.py` imports the reference in the build container
and writes `tests/golden/*.npz`; `tests/test_oracle_golden.py` replays them).

The restatement is deliberately *not* the reference's code shape:
  * routing uses a partition threshold + ordered tie fill instead of the
    reference's per-column rank insertion (src/router.py:89-115);
  * the varlen layout uses a stable counting sort instead of a cursor
    scatter (src/router.py:143-148);
  * attention walks key blocks (key-block-major, as the GPU does) and merges
    per-(query, block) partials with the same online-softmax algebra as
    SoftmaxState.update (src/attention.py:60-68).
All arithmetic is float64 unless the caller passes another dtype.
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "centroids",
    "key_conv_forward",
    "key_conv_backward",
    "random_conv_weights",
    "select_topk",
    "build_varlen",
    "build_plan",
    "validate_plan",
    "forward",
    "backward",
    "attention",
    "forward_rows",
    "backward_rows_dq",
    "backward_block",
    "visible_pairs",
    "plan_entries",
    "scored_candidates",
    "OraclePlan",
]


class OraclePlanError(ValueError):
    """Mirrors PlanValidationError (src/core.py:37-38) for oracle-side checks."""


class OraclePlan:
    """CSR routing plan, same fields as RoutingPlan (src/core.py:229-251)."""

    def __init__(self, topk_indices, counts, offsets, flat_queries):
        self.topk_indices = np.asarray(topk_indices, dtype=np.int32)
        self.counts = np.asarray(counts, dtype=np.int64)
        self.offsets = np.asarray(offsets, dtype=np.int64)
        self.flat_queries = np.asarray(flat_queries, dtype=np.int32)

    @property
    def n_blocks(self):
        return len(self.counts)


# --------------------------------------------------------------------------
# closed forms (tests/oracles.py:95-98, tests/test_router.py:169-172)
# --------------------------------------------------------------------------

def visible_pairs(N: int, B: int, k: int) -> int:
    """P = sum_i [min(k, i//B)*B + i%B + 1] (tests/oracles.py:95-98)."""
    i = np.arange(N, dtype=np.int64)
    return int((np.minimum(k, i // B) * B + i % B + 1).sum())


def plan_entries(N: int, B: int, k: int) -> int:
    """E = sum_i (1 + min(k, i//B)) (tests/test_router.py:169-172)."""
    i = np.arange(N, dtype=np.int64)
    return int((1 + np.minimum(k, i // B)).sum())


def scored_candidates(N: int, B: int) -> int:
    """R = sum_i i//B: (query, strictly-past block) pairs the router scores."""
    i = np.arange(N, dtype=np.int64)
    return int((i // B).sum())


# --------------------------------------------------------------------------
# stage 1: centroids (src/router.py:32-46) and key conv (src/keyconv.py)
# --------------------------------------------------------------------------

def centroids(K, B: int):
    """Per-block mean over the actual (ragged) block length.

    Follows compute_centroids (src/router.py:39-43): sum of the block's rows
    divided by min(B, N - jB). Returns (centroids [n,d], lengths [n] int64).
    """
    K = np.asarray(K)
    N, d = K.shape
    n = -(-N // B)
    pad = n * B - N
    Kp = np.concatenate([K, np.zeros((pad, d), K.dtype)]) if pad else K
    sums = Kp.reshape(n, B, d).sum(axis=1)
    lengths = np.minimum(B, N - np.arange(n) * B).astype(np.int64)
    return sums / lengths[:, None].astype(K.dtype), lengths


def _sigmoid(x):
    # overflow-safe two-branch sigmoid, as src/keyconv.py:50-56
    e = np.exp(-np.abs(x))
    return np.where(x >= 0, 1.0 / (1.0 + e), e / (1.0 + e))


def _conv_preact(K, W):
    # a_t = sum_l W[l] * K[t-l], zero left pad (src/keyconv.py:59-67)
    N = K.shape[0]
    a = np.zeros_like(K)
    for lag in range(min(W.shape[0], N)):
        a[lag:] += W[lag] * K[: N - lag]
    return a


def key_conv_forward(K, W):
    """K' = K + silu(conv(K)) (src/keyconv.py:70-78)."""
    K = np.asarray(K)
    W = np.asarray(W, dtype=K.dtype)
    a = _conv_preact(K, W)
    return K + a * _sigmoid(a)


def key_conv_backward(K, W, dK_out):
    """(dK, dW) of key_conv_forward (src/keyconv.py:81-104)."""
    K = np.asarray(K)
    W = np.asarray(W, dtype=K.dtype)
    N = K.shape[0]
    a = _conv_preact(K, W)
    s = _sigmoid(a)
    g = dK_out * (s * (1.0 + a * (1.0 - s)))
    dK = np.array(dK_out, copy=True)
    dW = np.zeros_like(W)
    for lag in range(min(W.shape[0], N)):
        dW[lag] = (g[lag:] * K[: N - lag]).sum(axis=0)
        dK[: N - lag] += W[lag] * g[lag:]
    return dK, dW


def random_conv_weights(width: int, d: int, seed: int):
    """U(-1/sqrt(width), 1/sqrt(width)) seeded, as random_kernel (src/keyconv.py:43-47)."""
    rng = np.random.default_rng(seed)
    bound = 1.0 / np.sqrt(width)
    return rng.uniform(-bound, bound, size=(width, d))


# --------------------------------------------------------------------------
# stage 2: top-k routing (src/router.py:49-120, src/reference.py:98-124)
# --------------------------------------------------------------------------

def _topk_rows(scores, own, k):
    """Top-k strictly-past blocks per row with ties to the lower index.

    scores: [r, n] float64, own: [r] own block ids. Candidates are j < own
    (src/router.py:92). Returns a boolean [r, n] selection mask.
    """
    r, n = scores.shape
    cols = np.arange(n)[None, :]
    past = cols < own[:, None]
    masked = np.where(past, scores, -np.inf)
    sel = np.zeros((r, n), dtype=bool)
    few = own <= k                       # every past block fits: take them all
    sel[few] = past[few]
    many = ~few
    if many.any():
        m = masked[many]
        # k-th largest value per row = threshold t
        t = -np.partition(-m, k - 1, axis=1)[:, k - 1]
        gt = m > t[:, None]
        eq = m == t[:, None]
        need = k - gt.sum(axis=1)
        # ties at the threshold resolve to the lower block index
        # (src/router.py:95-98; tests/test_router.py:91-98)
        fill = eq & (np.cumsum(eq, axis=1) <= need[:, None])
        sel[many] = gt | fill
    return sel


def select_topk(Q, cents, B: int, k: int, row_chunk: int = 2048):
    """Index matrix [N, k+1] int32: own block + top-k past blocks, ascending,
    -1 tail (src/router.py:116-119). Scores are the unscaled q . centroid
    (src/attention.py:312 routes with raw Q) evaluated in float64."""
    Q = np.asarray(Q, dtype=np.float64)
    cents = np.asarray(cents, dtype=np.float64)
    N = Q.shape[0]
    n = cents.shape[0]
    out = np.full((N, k + 1), -1, dtype=np.int32)
    for r0 in range(0, N, row_chunk):
        r1 = min(r0 + row_chunk, N)
        own = np.arange(r0, r1) // B
        sel = _topk_rows(Q[r0:r1] @ cents.T, own, k)
        sel[np.arange(r1 - r0), own] = True          # own block always attended
        cnt = sel.sum(axis=1)
        rr, cc = np.nonzero(sel)                      # row-major => ascending ids
        slot = np.arange(len(cc)) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        out[r0 + rr, slot] = cc
    return out


# --------------------------------------------------------------------------
# stage 3: varlen layout (src/router.py:123-154)
# --------------------------------------------------------------------------

def build_varlen(topk_indices, n_blocks: int) -> OraclePlan:
    """Key-block-major CSR via a stable counting sort over (block, query)."""
    idx = np.asarray(topk_indices)
    if idx.size and (idx.min() < -1 or idx.max() >= n_blocks):
        raise OraclePlanError("index entries out of range")  # src/router.py:134-138
    N, w = idx.shape
    rows = np.repeat(np.arange(N, dtype=np.int64), w)
    cols = idx.reshape(-1).astype(np.int64)
    keep = cols >= 0
    rows, cols = rows[keep], cols[keep]
    order = np.argsort(cols, kind="stable")           # rows already ascending
    counts = np.bincount(cols, minlength=n_blocks).astype(np.int64)
    offsets = np.concatenate(([0], np.cumsum(counts)[:-1])).astype(np.int64)
    return OraclePlan(idx.astype(np.int32), counts, offsets, rows[order].astype(np.int32))


def build_plan(Q, K, B: int, k: int) -> OraclePlan:
    """centroids -> top-k -> varlen (src/router.py:157-161)."""
    c, _ = centroids(np.asarray(K, dtype=np.float64), B)
    return build_varlen(select_topk(Q, c, B, k), c.shape[0])


def validate_plan(plan: OraclePlan, N: int, B: int) -> None:
    """Invariants of validate_plan (src/core.py:254-296), vectorised."""
    n = -(-N // B)
    idx = plan.topk_indices
    if idx.ndim != 2 or idx.shape[0] != N:
        raise OraclePlanError("topk shape")
    if plan.counts.shape != (n,) or plan.offsets.shape != (n,):
        raise OraclePlanError("counts/offsets length")
    if np.any(plan.counts < 0):
        raise OraclePlanError("negative count")
    if not np.array_equal(plan.offsets, np.concatenate(([0], np.cumsum(plan.counts)[:-1]))):
        raise OraclePlanError("offsets not exclusive prefix sum")
    total = int(plan.counts.sum())
    if len(plan.flat_queries) != total or int((idx >= 0).sum()) != total:
        raise OraclePlanError("entry count")
    valid = idx >= 0
    if valid.any() and idx[valid].max() >= n:
        raise OraclePlanError("block out of range")
    own = (np.arange(N) // B)[:, None]
    if np.any(valid & (idx > own)):
        raise OraclePlanError("causality")
    s = np.sort(np.where(valid, idx, -1 - np.arange(idx.shape[1])[None, :]), axis=1)
    if np.any(s[:, 1:] == s[:, :-1]):
        raise OraclePlanError("duplicate block in a row")
    blk = np.repeat(np.arange(n), plan.counts)
    fq = plan.flat_queries.astype(np.int64)
    if total:
        same = blk[1:] == blk[:-1]
        if np.any(same & (np.diff(fq) <= 0)):
            raise OraclePlanError("slice not strictly ascending")
        if np.any(fq < blk * B) or np.any(fq >= N):
            raise OraclePlanError("query outside [jB, N)")


# --------------------------------------------------------------------------
# attention forward / backward (src/attention.py:96-182, :195-302)
# --------------------------------------------------------------------------

def _block_slice(plan, j):
    o = int(plan.offsets[j])
    return plan.flat_queries[o : o + int(plan.counts[j])].astype(np.int64)


def forward(Q, K, V, plan: OraclePlan, B: int, dtype=np.float64):
    """Plan-driven attention: O [N,d], LSE [N] (natural log, scaled scores).

    Key-block-major walk; each (query, block) contributes one softmax
    partial merged with the online-softmax rule of SoftmaxState.update
    (src/attention.py:60-68) and finalised as O = acc/l, L = m + log l
    (src/attention.py:70-74). Token-causal mask key > query
    (src/attention.py:127-133); Q is pre-scaled by 1/sqrt(d)
    (src/attention.py:159-160).
    """
    Q = np.asarray(Q, dtype=dtype)
    K = np.asarray(K, dtype=dtype)
    V = np.asarray(V, dtype=dtype)
    N, d = Q.shape
    Qs = Q * (1.0 / np.sqrt(d))
    m = np.full(N, -np.inf, dtype=dtype)
    l = np.zeros(N, dtype=dtype)
    acc = np.zeros((N, d), dtype=dtype)
    for j in range(plan.n_blocks):
        rows = _block_slice(plan, j)
        if rows.size == 0:
            continue
        k0, k1 = j * B, min(j * B + B, N)
        S = Qs[rows] @ K[k0:k1].T
        S = np.where(np.arange(k0, k1)[None, :] > rows[:, None], -np.inf, S)
        mb = S.max(axis=1)
        m_new = np.maximum(m[rows], mb)
        p = np.exp(S - m_new[:, None])
        alpha = np.exp(m[rows] - m_new)
        l[rows] = l[rows] * alpha + p.sum(axis=1)
        acc[rows] = acc[rows] * alpha[:, None] + p @ V[k0:k1]
        m[rows] = m_new
    return acc / l[:, None], m + np.log(l)


def backward(Q, K, V, O, dO, lse, plan: OraclePlan, B: int, dtype=np.float64):
    """(dQ, dK, dV) with the plan frozen: recompute P = exp(S - L)
    (src/attention.py:229), dV += P^T dO, dP = dO V^T, dS = P (dP - D),
    dK += dS^T Q_scaled, dQ += dS K (src/attention.py:230-234), D =
    rowsum(dO*O) (src/attention.py:266), dQ scaled by 1/sqrt(d) at the end
    (src/attention.py:299)."""
    Q, K, V, O, dO = (np.asarray(x, dtype=dtype) for x in (Q, K, V, O, dO))
    lse = np.asarray(lse, dtype=dtype)
    N, d = Q.shape
    scale = 1.0 / np.sqrt(d)
    Qs = Q * scale
    D = (dO * O).sum(axis=1)
    dQ = np.zeros((N, d), dtype=np.float64)
    dK = np.zeros((N, d), dtype=dtype)
    dV = np.zeros((N, d), dtype=dtype)
    for j in range(plan.n_blocks):
        rows = _block_slice(plan, j)
        if rows.size == 0:
            continue
        k0, k1 = j * B, min(j * B + B, N)
        S = Qs[rows] @ K[k0:k1].T
        S = np.where(np.arange(k0, k1)[None, :] > rows[:, None], -np.inf, S)
        P = np.exp(S - lse[rows][:, None])
        dV[k0:k1] += P.T @ dO[rows]
        dS = P * (dO[rows] @ V[k0:k1].T - D[rows][:, None])
        dK[k0:k1] += dS.T @ Qs[rows]
        dQ[rows] += dS @ K[k0:k1]           # rows unique within a slice
    return (dQ * scale).astype(dtype), dK, dV


def attention(Q, K, V, B: int, k: int, conv_W=None):
    """End-to-end oracle of moba_attention (src/attention.py:305-314), with
    the optional key conv applied to K first (src/cli.py:277-278).
    Returns (O, LSE, plan, K_used)."""
    Kf = np.asarray(K, dtype=np.float64)
    if conv_W is not None:
        Kf = key_conv_forward(Kf, np.asarray(conv_W, dtype=np.float64))
    plan = build_plan(Q, Kf, B, k)
    O, L = forward(Q, Kf, V, plan, B)
    return O, L, plan, Kf


# --------------------------------------------------------------------------
# row / block restrictions of forward and backward, for sampled checks at
# sizes where the whole-head oracle is too slow (512K): the same algebra as
# forward / backward above, restricted to chosen query rows or key blocks
# --------------------------------------------------------------------------

def _row_keys(i: int, blocks, B: int, N: int):
    """Visible keys of query i over its plan blocks: whole blocks, own block
    up to i (token-causal mask key > query, src/attention.py:127-133)."""
    ks = [np.arange(j * B, min(j * B + B, N, i + 1)) for j in blocks if j >= 0]
    return np.concatenate(ks) if ks else np.zeros(0, dtype=np.int64)


def forward_rows(Q, K, V, rows, topk_rows, B: int):
    """O [r, d], LSE [r] for the query rows `rows` given their plan rows
    (topk_rows [r, width], -1 tail): one softmax over all visible keys of the
    row's blocks, equal to merging the per-block partials
    (SoftmaxState.update/finalize, src/attention.py:60-74)."""
    Q, K, V = (np.asarray(x, dtype=np.float64) for x in (Q, K, V))
    N, d = Q.shape
    scale = 1.0 / np.sqrt(d)
    O = np.zeros((len(rows), d))
    L = np.zeros(len(rows))
    for r, i in enumerate(rows):
        ks = _row_keys(int(i), topk_rows[r], B, N)
        s = (Q[i] * scale) @ K[ks].T
        m = s.max()
        p = np.exp(s - m)
        O[r] = p @ V[ks] / p.sum()
        L[r] = m + np.log(p.sum())
    return O, L


def backward_rows_dq(Q, K, V, O_rows, dO, L_rows, rows, topk_rows, B: int):
    """dQ rows: dQ_i = scale * sum_k P_ik (dP_ik - D_i) K_k with P = exp(S -
    L), dP = dO V^T, D_i = dO_i . O_i (src/attention.py:229-234, :266,
    :299)."""
    Q, K, V, dO = (np.asarray(x, dtype=np.float64) for x in (Q, K, V, dO))
    N, d = Q.shape
    scale = 1.0 / np.sqrt(d)
    dQ = np.zeros((len(rows), d))
    for r, i in enumerate(rows):
        ks = _row_keys(int(i), topk_rows[r], B, N)
        P = np.exp((Q[i] * scale) @ K[ks].T - L_rows[r])
        dS = P * (dO[i] @ V[ks].T - dO[i] @ O_rows[r])
        dQ[r] = scale * (dS @ K[ks])
    return dQ


def backward_block(Q, K, V, dO, j: int, queries, O_q, L_q, B: int):
    """(dK_j, dV_j) [len_j, d] of key block j from the queries attending it
    (its flat slice) with their O and LSE: dV_j = P^T dO, dK_j = dS^T
    Q_scaled (src/attention.py:230-233)."""
    Q, K, V, dO = (np.asarray(x, dtype=np.float64) for x in (Q, K, V, dO))
    N, d = Q.shape
    scale = 1.0 / np.sqrt(d)
    k0, k1 = j * B, min(j * B + B, N)
    q = np.asarray(queries, dtype=np.int64)
    S = (Q[q] * scale) @ K[k0:k1].T
    S = np.where(np.arange(k0, k1)[None, :] > q[:, None], -np.inf, S)
    P = np.exp(S - np.asarray(L_q)[:, None])
    Dq = (dO[q] * np.asarray(O_q)).sum(axis=1)
    dS = P * (dO[q] @ V[k0:k1].T - Dq[:, None])
    return dS.T @ (Q[q] * scale), P.T @ dO[q]
