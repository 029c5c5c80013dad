// Tensor-core top-k routing with an exactness guard (select_topk,
// src/router.py:49-120, tensor-core mode).
//
// Scores S = Q (C_hi + C_lo)^T on tcgen05: the fp32 centroids are split into
// two bf16 terms (|c - c_hi - c_lo| <= 2^-16 |c|), Q is bf16 (exact), fp32
// accumulation in TMEM.
//
// Persistent kernel, one CTA per SM. A work unit is T consecutive 128-query
// tiles of one head (T = 3 at d = 64, 2 at d = 128); every 128-centroid chunk
// is loaded once per unit (TMA, CS smem stages) and multiplied, as two
// N = 64 sub-chunks, into each tile's own double-buffered TMEM columns, so the
// centroid traffic is shared by T tiles. Units are dealt round robin in
// longest-first order (the last tiles of a head see the most past blocks).
//
// Warps (32 x (1 + 5T) threads):
//   0        TMA loads of the centroid chunks through the stages
//   1 .. T   MMA issue, one warp per tile (its Q tile load, then its score
//            sub-chunks, warp-uniform with one elected lane): the tiles do
//            not wait for each other, only for their own buffers
//   T+1 ..   selection: 4 warps per tile (TMEM lane quadrant = warp % 4),
//            one query row per thread over every chunk of the row.
//
// Selection keeps a sorted list of LS = top_k + 2 (+ 3) packed 32-bit keys per
// row: the order-preserving bits of the tensor-core score with the low
// `idx_bits` replaced by (2^idx_bits - 1 - j), so one unsigned compare
// orders by (truncated score desc, block index asc) and inserting a key
// costs two IMNMX per list slot. A 16-candidate sub-group is filtered with
// one FSETP per candidate against the list's threshold; only when some lane
// of the warp has a hit are the 16 scores staged (lane-private smem) and the
// hits inserted, one per lane per round.
//
// Exactness (the output is bitwise the fp32 router's, route_topk_fp32_kernel,
// whose scores are the fp32 FFMA chain over d): with
//   E(row) = (kEps(D) + 2^(idx_bits - 22)) * |q| * max_j |c_j|
// bounding |key score - fp32 score| (split error, tensor-core accumulation,
// FFMA chain, key truncation; x2 margins) and s_u the key score of list
// entry u,
//   s_{k-1} - s_k    > 2E -> the listed top k IS the fp32 top k;
//   s_{k-1} - s_{LS-1} > 2E -> the fp32 top k lies inside the LS listed
//                            entries: the warp rescoring them with the fp32
//                            chain (one lane per entry) and reselects;
//   otherwise              -> the row's 128-query tile is listed for the exact
//                            fp32 router (route_topk_fp32_kernel, tile-list
//                            mode), which routes the whole tile again.
#include "common.cuh"
#include "sm100.cuh"
#include <algorithm>
#include <type_traits>

namespace moba {
namespace rtc {

constexpr int kM = 128;            // queries per tile (TMEM lanes)
constexpr int kN = 128;            // centroids per chunk (MMA N)
constexpr int kSplits = 2;         // bf16 hi + lo terms of the fp32 centroids
constexpr int kW = 64;             // score columns per TMEM buffer (MMA N of one sub-chunk)

// TT: query tiles per unit — 4 (21 warps, more selection warps in flight
// per SM) at d = 64 (the launch table in launch_route_tc), 2 (11 warps) at
// d = 128; 3 (16 warps) is kept for the A/B record
template <int D, int TT = (D == 64) ? 3 : 2>
struct Geo {
    static constexpr int T = TT;
    static constexpr int NBUF = (D == 64) ? 2 : 4;       // TMEM score buffers per tile
    static constexpr int CS = (D == 64) ? 3 : 2;         // centroid chunk smem stages
    static constexpr int kSelWarps = 4 * T;
    static constexpr int kSel0 = 1 + T;                  // first selection warp
    static constexpr int kThreads = 32 * (kSel0 + kSelWarps);
    static constexpr uint32_t kQ = kM * D * 2;           // one query tile
    static constexpr uint32_t kCterm = kN * D * 2;
    static constexpr uint32_t kC = kSplits * kCterm;     // one chunk stage
    static constexpr uint32_t kStgWarp = 32 * 128;       // 32 scores per lane (16-B chunks swizzled by lane)
    static constexpr uint32_t kBars = 512;
    static constexpr uint32_t kSmem = 1024 + T * kQ + CS * kC + kSelWarps * kStgWarp + kBars;
    static_assert(T * NBUF * kW <= 512, "the score buffers fit TMEM");
    static_assert(kSmem <= 232448, "shared memory");
    // |s_tc - s_fp32| <= kEps * |q| * max|c|, with
    //   split:       2^-16 (two bf16 terms)
    //   tc accum.:   2 * (kSplits * D / 16 + 1) * 2^-23 (per K=16 MMA step, truncating)
    //   fp32 chain:  D * 2^-24 (sequential FFMA over d)
    // and a 2x safety margin
    static constexpr float kEps = 2.0f * (1.52587890625e-05f + 2.0f * (kSplits * D / 16 + 1) * 1.1920928955078125e-07f +
                                          D * 5.9604644775390625e-08f);
};

struct Bars {
    uint64_t c_full[3], c_empty[3], q_full[4], q_empty[4], s_full[4][4], s_free[4][4];
    uint32_t tmem;
};

// order-preserving unsigned image of an fp32 score (and its inverse)
MOBA_DEV uint32_t okey(float s) {
    const uint32_t u = __float_as_uint(s);
    return u ^ ((uint32_t)((int32_t)u >> 31) | 0x80000000u);
}
MOBA_DEV float okey_decode(uint32_t k) { return __uint_as_float((k & 0x80000000u) ? (k ^ 0x80000000u) : ~k); }
// truncated score of a list key (a lower bound of the score it was built
// from); -inf for the empty key 0
MOBA_DEV float key_score(uint32_t k, uint32_t imask) { return k == 0u ? -INFINITY : okey_decode(k & ~imask); }

// sorted (descending) insertion of x: slot u becomes max(ts[u], min(ts[u-1], x))
// (keep, take x, or shift down) — every slot reads the old list, so the
// network is two IMNMX deep instead of a chain through the list; x = 0 is a
// no-op
template <int LS>
MOBA_DEV void key_insert(uint32_t (&ts)[LS], uint32_t x) {
    uint32_t nw[LS];
    nw[0] = max(ts[0], x);
#pragma unroll
    for (int u = 1; u < LS; ++u) nw[u] = max(ts[u], min(ts[u - 1], x));
#pragma unroll
    for (int u = 0; u < LS; ++u) ts[u] = nw[u];
}

// sorted insertion of two keys x >= y (merge of a 2-list): slot u becomes the
// (u+1)-th largest of the union, max(ts[u], min(ts[u-1], x), min(ts[u-2], y));
// one VIMNMX3 and two IMNMX per slot, all reading the old list
template <int LS>
MOBA_DEV void key_insert2(uint32_t (&ts)[LS], uint32_t x, uint32_t y) {
    uint32_t nw[LS];
    nw[0] = max(ts[0], x);
    if (LS > 1) nw[1] = max(max(ts[1], min(ts[0], x)), y);
#pragma unroll
    for (int u = 2; u < LS; ++u) nw[u] = max(max(ts[u], min(ts[u - 1], x)), min(ts[u - 2], y));
#pragma unroll
    for (int u = 0; u < LS; ++u) ts[u] = nw[u];
}

// candidate (s, j) with j larger than every listed index: after every entry
// with score >= s (ties keep the lower index first)
template <int LS>
MOBA_DEV void list_insert(float (&ts)[LS], int (&ti)[LS], float s, int j) {
    bool ge[LS];
#pragma unroll
    for (int u = 0; u < LS; ++u) ge[u] = ts[u] >= s;
#pragma unroll
    for (int u = LS - 1; u >= 1; --u) {
        const float ns = ge[u - 1] ? s : ts[u - 1];
        const int ni = ge[u - 1] ? j : ti[u - 1];
        ts[u] = ge[u] ? ts[u] : ns;
        ti[u] = ge[u] ? ti[u] : ni;
    }
    ts[0] = ge[0] ? ts[0] : s;
    ti[0] = ge[0] ? ti[0] : j;
}

// the same chain with q in registers
template <int D>
MOBA_DEV float exact_score(const float (&q)[D], const float* __restrict__ c) {
    float acc = 0.f;
#pragma unroll
    for (int dd = 0; dd < D; dd += 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(c + dd));
        acc = fmaf(q[dd], v.x, acc);
        acc = fmaf(q[dd + 1], v.y, acc);
        acc = fmaf(q[dd + 2], v.z, acc);
        acc = fmaf(q[dd + 3], v.w, acc);
    }
    return acc;
}

// (score desc, index asc)
MOBA_DEV bool better(float a, int ia, float b, int ib) { return a > b || (a == b && ia < ib); }

// sort block ids ascending, append the own block, pad with -1
template <int KMAX>
MOBA_DEV void write_row(int32_t* out, int (&res)[KMAX], int top_k, int own, int width) {
#pragma unroll
    for (int u = 0; u < KMAX; ++u)
        if (u >= top_k) res[u] = 0x7fffffff;
#pragma unroll
    for (int p = 0; p < KMAX; ++p)
#pragma unroll
        for (int u = (p & 1); u + 1 < KMAX; u += 2) {
            const int x = res[u], y = res[u + 1];
            res[u] = min(x, y);
            res[u + 1] = max(x, y);
        }
    int nvalid = 0;
#pragma unroll
    for (int u = 0; u < KMAX; ++u)
        if (res[u] != 0x7fffffff) out[nvalid++] = res[u];
    out[nvalid] = own;
    for (int s = nvalid + 1; s < width; ++s) out[s] = -1;
}



// m += bit when s >= thr: FSETP + a predicated IMAD (one * bit + m, `one` a
// register ptxas cannot prove to be 1, so the add stays an IMAD on the FMA
// pipe instead of an IADD3 / SEL on the ALU)
MOBA_DEV void filter_add(uint32_t& m, float s, float thr, uint32_t one, uint32_t bit) {
    asm("{\n\t.reg .pred p;\n\tsetp.ge.f32 p, %1, %2;\n\t@p mad.lo.u32 %0, %3, %4, %0;\n\t}\n"
        : "+r"(m)
        : "f"(s), "f"(thr), "r"(one), "r"(bit));
}

// the lane's next pending hit of the group: its staged score (lane-private
// row at stg, 16-B chunks XOR-swizzled by sx4) and its key-index field; the
// no-op key source (score unused, idx 0 with key 0) when none is left
MOBA_DEV bool next_hit(uint32_t& m, uint32_t stg, uint32_t sx4, float& s, uint32_t& e) {
    if (m == 0u) return false;
    e = (uint32_t)__ffs(m) - 1u;
    m &= m - 1u;
    asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(s) : "r"(stg | ((e << 2) ^ sx4)));
    return true;
}

// exact fp32 score from global memory (the fp32 router's chain)
template <int D>
MOBA_DEV float exact_score_g(const __nv_bfloat16* __restrict__ q, const float* __restrict__ c) {
    float acc = 0.f;
#pragma unroll
    for (int dd = 0; dd < D; dd += 8) {
        float x[8];
        ld8f(q + dd, x);
        const float4 v0 = __ldg(reinterpret_cast<const float4*>(c + dd));
        const float4 v1 = __ldg(reinterpret_cast<const float4*>(c + dd) + 1);
        const float cv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) acc = fmaf(x[e], cv[e], acc);
    }
    return acc;
}

template <int D, int KMAX, int TT, int LX>
__global__ void __launch_bounds__(Geo<D, TT>::kThreads, 1)
route_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_c,
                const __nv_bfloat16* __restrict__ Q, const float* __restrict__ cent, const float* __restrict__ cmax2,
                int64_t N, int B, int top_k, int64_t split_rows, int kv_group, int bh, int n_tiles, int n_groups,
                int idx_bits, int32_t* __restrict__ topk, int* __restrict__ recheck) {
    using namespace sm100;
    using G = Geo<D, TT>;
    constexpr int T = G::T, NBUF = G::NBUF, CS = G::CS;
    // list length k + LX: LX = 2 while a row has <= ~2K candidates, 3 from
    // 256K tokens, whose denser score tails leave more rows undecided with a
    // short list (route_topk_launch)
    constexpr int LS_EXTRA = LX;
    constexpr int LS = (KMAX + LS_EXTRA < 32) ? KMAX + LS_EXTRA : 32;
    constexpr int SL = D / 64;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sq = smem_u32(smem);
    const uint32_t sc = sq + T * G::kQ;
    const uint32_t sstg = sc + CS * G::kC;
    Bars* bars = reinterpret_cast<Bars*>(smem + T * G::kQ + CS * G::kC + G::kSelWarps * G::kStgWarp);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n_blocks = (int)((N + B - 1) / B);
    const int width = top_k + 1;
    const int total = bh * n_groups;
    const int n_my = total > (int)blockIdx.x ? (total - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    // unit i of this CTA -> (head, tile group), longest first
    auto unit_h = [&](int i) { return (int)(((int)blockIdx.x + i * (int)gridDim.x) % bh); };
    auto unit_g = [&](int i) { return n_groups - 1 - ((int)blockIdx.x + i * (int)gridDim.x) / bh; };
    // 64-centroid sub-chunks tile t needs: candidates j < own <= own of its last row
    auto tile_nsub = [&](int t) -> int {
        if (t >= n_tiles) return 0;
        const int mo = (int)((min64((int64_t)(t + 1) * kM, N) - 1) / B);
        return (mo + kW - 1) / kW;
    };
    auto unit_nch = [&](int i) {
        const int t = min(unit_g(i) * T + T - 1, n_tiles - 1);
        return (tile_nsub(t) + 1) / 2;
    };

    if (warp == 0) tmem_alloc(&bars->tmem, 512);
    if (tid == 0) {
        for (int i = 0; i < CS; ++i) {
            mbar_init(&bars->c_full[i], 1);
            mbar_init(&bars->c_empty[i], T);
        }
        for (int t = 0; t < T; ++t) {
            mbar_init(&bars->q_full[t], 1);
            mbar_init(&bars->q_empty[t], 1 + 4);
            for (int b = 0; b < NBUF; ++b) {
                mbar_init(&bars->s_full[t][b], 1);
                mbar_init(&bars->s_free[t][b], 4);
            }
        }
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem;

    if (warp == 0) {
        // ------------------------------------------------------------ centroid loader
        int gl = 0;
        for (int i = 0; i < n_my; ++i) {
            const int nch = unit_nch(i);
            const int64_t hk = unit_h(i) / kv_group;
            for (int c = 0; c < nch; ++c, ++gl) {
                const int st = gl % CS;
                if (gl >= CS) mbar_wait_sleep(&bars->c_empty[st], ((gl / CS) - 1) & 1);
                if (lane == 0) {
                    mbar_expect_tx(&bars->c_full[st], G::kC);
#pragma unroll
                    for (int t = 0; t < kSplits; ++t)
#pragma unroll
                        for (int sl = 0; sl < SL; ++sl)
                            tma_load_2d(sc + st * G::kC + t * G::kCterm + sl * kN * 128, &tm_c, sl * 64,
                                        (int)(t * split_rows + hk * n_blocks + (int64_t)c * kN), &bars->c_full[st]);
                }
                __syncwarp();
            }
        }
    } else if (warp < G::kSel0) {
        // ------------------------------------------------------------ MMA issuer of tile warp - 1
        // (its own Q tile load, then S sub-chunks into the tile's buffers;
        // a chunk stage is released once every tile's MMAs have read it)
        const int tt = warp - 1;
        const uint32_t idesc = idesc_bf16(kM, kW, false, false);
        int gm = 0, qc = 0, scnt[NBUF];
#pragma unroll
        for (int b = 0; b < NBUF; ++b) scnt[b] = 0;
        for (int i = 0; i < n_my; ++i) {
            const int h = unit_h(i), t = unit_g(i) * T + tt;
            const int nch = unit_nch(i);
            const int nsub = tile_nsub(t);
            if (nsub > 0) {
                if (qc > 0) mbar_wait_sleep(&bars->q_empty[tt], (qc - 1) & 1);
                if (lane == 0) {
                    mbar_expect_tx(&bars->q_full[tt], G::kQ);
#pragma unroll
                    for (int sl = 0; sl < SL; ++sl)
                        tma_load_2d(sq + tt * G::kQ + sl * kM * 128, &tm_q, sl * 64,
                                    (int)((int64_t)h * N + (int64_t)t * kM), &bars->q_full[tt]);
                }
                __syncwarp();
            }
            for (int c = 0; c < nch; ++c) {
                const int st = (gm + c) % CS;
                mbar_wait_sleep(&bars->c_full[st], ((gm + c) / CS) & 1);
                if (2 * c >= nsub) {
                    if (lane == 0) mbar_arrive(&bars->c_empty[st]);
                    __syncwarp();
                    continue;
                }
                if (c == 0) mbar_wait_sleep(&bars->q_full[tt], qc & 1);
                const uint32_t cb = sc + st * G::kC;
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    const int sub = 2 * c + hf;
                    if (sub >= nsub) continue;
#pragma unroll
                    for (int b = 0; b < NBUF; ++b) {
                        if ((sub % NBUF) != b) continue;
                        if (scnt[b] > 0) mbar_wait_sleep(&bars->s_free[tt][b], (scnt[b] - 1) & 1);
                        tc_fence_after();
                        const uint32_t dst = tmem + (uint32_t)((tt * NBUF + b) * kW);
#pragma unroll
                        for (int t2 = 0; t2 < kSplits; ++t2)
#pragma unroll
                            for (int kk = 0; kk < D / 16; ++kk) {
                                const int sl = kk >> 2, ke = (kk & 3) * 16;
                                umma_bf16_w(dst, desc_kmajor(sq + tt * G::kQ + sl * kM * 128, ke),
                                            desc_kmajor(cb + t2 * G::kCterm + sl * kN * 128 + hf * kW * 128, ke),
                                            idesc, t2 > 0 || kk > 0);
                            }
                        umma_commit_w(&bars->s_full[tt][b]);
                        ++scnt[b];
                    }
                }
                umma_commit_w(&bars->c_empty[st]);
                if (2 * c + 2 >= nsub) {
                    umma_commit_w(&bars->q_empty[tt]);
                    ++qc;
                }
            }
            gm += nch;
        }
    } else {
        // ------------------------------------------------------------ selection
        const int sw = warp - G::kSel0, tt = sw >> 2, quad = warp & 3;
        const int row = 32 * quad + lane;
        const uint32_t lane_off = (uint32_t)(32 * quad) << 16;
        const uint32_t stg = sstg + sw * G::kStgWarp + lane * 128;
        const uint32_t sxor = (uint32_t)(lane & 7), sx4 = sxor << 4;
        const uint32_t imask = (1u << idx_bits) - 1u;
        const float gstep = ldexpf(1.f, idx_bits - 22);   // key grid step / 2^exponent (x2 margin)
        const uint32_t one = (uint32_t)min(n_tiles, 1);      // 1 (n_tiles >= 1), opaque to ptxas
        int qcnt = 0, scnt[NBUF];
#pragma unroll
        for (int b = 0; b < NBUF; ++b) scnt[b] = 0;
        for (int i = 0; i < n_my; ++i) {
            const int h = unit_h(i), t = unit_g(i) * T + tt;
            if (t >= n_tiles) continue;
            const int64_t hk = h / kv_group;
            const int64_t r0 = (int64_t)t * kM;
            const int64_t my_i = r0 + row;
            const bool valid = my_i < N;
            const int own = valid ? (int)(my_i / B) : 0;
            const int nsub = tile_nsub(t);
            uint32_t ts[LS];
#pragma unroll
            for (int u = 0; u < LS; ++u) ts[u] = 0u;
            float qn = 0.f;
            if (nsub > 0) {
                mbar_wait(&bars->q_full[tt], qcnt & 1);
                ++qcnt;
#pragma unroll
                for (int cg = 0; cg < D / 8; ++cg) {
                    const int sl = cg >> 3, ch = cg & 7;
                    const int4 raw = lds128i(sq + tt * G::kQ + sl * kM * 128 + row * 128 + ((ch ^ (row & 7)) << 4));
                    const uint32_t u4[4] = {(uint32_t)raw.x, (uint32_t)raw.y, (uint32_t)raw.z, (uint32_t)raw.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 f = unpack_bf16(u4[e]);
                        qn = fmaf(f.x, f.x, fmaf(f.y, f.y, qn));
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->q_empty[tt]);
                const int wown = __reduce_max_sync(0xffffffffu, own);
                float thr = -INFINITY;
                // a candidate whose key could never reach within the guard's
                // margin of the current k-th score (lo) is irrelevant to the
                // final decision: lo only rises, so s + grid(s) < lo - e2 now
                // stays true, and such a row's status is the same with or
                // without it listed. Filtering against max(list tail,
                // lo - e2 - grid) instead of the list tail alone drops ~1/3
                // of the insertions (top_k == KMAX keeps the index static).
                const float e2g = 2.f * G::kEps * sqrtf(qn) * sqrtf(__ldg(cmax2 + hk));
                for (int sub = 0; sub < nsub; ++sub) {
                    const int b = sub % NBUF;
#pragma unroll
                    for (int bb = 0; bb < NBUF; ++bb)
                        if (bb == b) {
                            mbar_wait(&bars->s_full[tt][bb], scnt[bb] & 1);
                            ++scnt[bb];
                        }
                    tc_fence_after();
                    const int ng = max(0, min(kW / 32, (wown - sub * kW + 31) / 32));
                    const uint32_t scol = tmem + (uint32_t)((tt * NBUF + b) * kW) + lane_off;
                    if (ng == 0) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&bars->s_free[tt][b]);
                    }
                    for (int g = 0; g < ng; ++g) {
                        const int j0 = sub * kW + 32 * g;
                        const int lim = max(0, min(32, own - j0));
                        const uint32_t jb = imask - (uint32_t)j0;
                        const bool warm = sub == 0 && g == 0 && __reduce_max_sync(0xffffffffu, lim) >= 12;
                        uint32_t m = 0;
                        // two 16-column halves keep the register peak low
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
                            float sv[16];
                            tmem_ld16(scol + 32 * g + 16 * hh, sv);
                            tmem_ld_wait();
                            if (g == ng - 1 && hh == 1) {
                                tc_fence_before();
                                __syncwarp();
                                if (lane == 0) mbar_arrive(&bars->s_free[tt][b]);
                            }
                            if (warm) {
                                // empty lists: insert the first 32 candidates unconditionally
#pragma unroll
                                for (int e = 0; e < 16; e += 2) {
                                    const uint32_t k0 = 16 * hh + e < lim
                                                            ? (okey(sv[e]) & ~imask) | (jb - (uint32_t)(16 * hh + e)) : 0u;
                                    const uint32_t k1 = 16 * hh + e + 1 < lim
                                                            ? (okey(sv[e + 1]) & ~imask) | (jb - (uint32_t)(16 * hh + e + 1)) : 0u;
                                    key_insert2<LS>(ts, max(k0, k1), min(k0, k1));
                                }
                            } else {
                                // hit bit e: one FSETP (ALU) and a predicated
                                // add of the bit (IMAD.IADD, FMA pipe) — the
                                // selection is ALU bound, and SEL + IADD3
                                // would put both halves on the ALU
                                uint32_t m0 = 0u, m1 = 0u;
#pragma unroll
                                for (int e = 0; e < 16; e += 2) {
                                    filter_add(m0, sv[e], thr, one, 1u << (16 * hh + e));
                                    filter_add(m1, sv[e + 1], thr, one, 1u << (16 * hh + e + 1));
                                }
                                m |= m0 + m1;
#pragma unroll
                                for (int e = 0; e < 16; e += 4)
                                    sts128(stg + ((((uint32_t)(16 * hh + e) >> 2) ^ sxor) << 4),
                                           make_uint4(__float_as_uint(sv[e]), __float_as_uint(sv[e + 1]),
                                                      __float_as_uint(sv[e + 2]), __float_as_uint(sv[e + 3])));
                            }
                        }
                        m &= lim >= 32 ? 0xffffffffu : (1u << max(lim, 0)) - 1u;
                        if (!warm && __any_sync(0xffffffffu, m != 0u)) {
                            // two hits per lane per round (a 2-key merge), the
                            // next round's scores loaded while this one merges
                            float s0 = 0.f, s1 = 0.f;
                            uint32_t e0 = 0u, e1 = 0u;
                            bool v0 = next_hit(m, stg, sx4, s0, e0);
                            bool v1 = next_hit(m, stg, sx4, s1, e1);
                            do {
                                float s2 = 0.f, s3 = 0.f;
                                uint32_t e2 = 0u, e3 = 0u;
                                const bool v2 = next_hit(m, stg, sx4, s2, e2);
                                const bool v3 = next_hit(m, stg, sx4, s3, e3);
                                const uint32_t k0 = v0 ? (okey(s0) & ~imask) | (jb - e0) : 0u;
                                const uint32_t k1 = v1 ? (okey(s1) & ~imask) | (jb - e1) : 0u;
                                key_insert2<LS>(ts, max(k0, k1), min(k0, k1));
                                v0 = v2;
                                v1 = v3;
                                s0 = s2;
                                s1 = s3;
                                e0 = e2;
                                e1 = e3;
                            } while (__any_sync(0xffffffffu, v0));
                        }
                        thr = key_score(ts[LS - 1], imask);
                        if (top_k == KMAX) {
                            const float lo_k = key_score(ts[KMAX - 1], imask);
                            thr = fmaxf(thr, lo_k - e2g - (fabsf(lo_k) + e2g) * 2.f * gstep);
                        }
                    }
                }
            }
            // ---------------------------------------------------------------- guard
            int res[KMAX];
#pragma unroll
            for (int u = 0; u < KMAX; ++u)
                res[u] = (u < top_k && ts[u] != 0u) ? (int)(imask - (ts[u] & imask)) : 0x7fffffff;
            int status = 0;
            if (valid && own > top_k) {
                // entries k-1 and k by a select chain (an indexed read would
                // send the whole list to local memory)
                uint32_t kk0 = 0u, kk1 = 0u;
#pragma unroll
                for (int u = 0; u < LS; ++u) {
                    uint32_t v;
                    asm volatile("mov.b32 %0, %1;\n" : "=r"(v) : "r"(ts[u]));
                    kk0 = (u == top_k - 1) ? v : kk0;
                    kk1 = (u == top_k) ? v : kk1;
                }
                // s_tc of a listed entry lies in [key score, key score + grid step);
                // every entry at or below position u has s_tc < upper(u)
                auto upper = [&](uint32_t key) {
                    const float v = key_score(key, imask);
                    return key == 0u ? -INFINITY : v + __uint_as_float(__float_as_uint(v) & 0x7f800000u) * gstep;
                };
                const float lo = key_score(kk0, imask);
                const float e2 = 2.f * G::kEps * sqrtf(qn) * sqrtf(__ldg(cmax2 + hk));
                if (!(lo - upper(kk1) > e2)) status = (lo - upper(ts[LS - 1]) > e2) ? 1 : 2;
            }
            // rows whose fp32 top k lies inside the list: the warp rescores
            // them one row at a time, lane u taking list entry u
            uint32_t rm = __ballot_sync(0xffffffffu, status == 1);
            while (rm != 0u) {
                const int r = __ffs(rm) - 1;
                rm &= rm - 1u;
                int cand = -1;
#pragma unroll
                for (int u = 0; u < LS; ++u) {
                    const uint32_t kv = __shfl_sync(0xffffffffu, ts[u], r);
                    if (lane == u && kv != 0u) cand = (int)(imask - (kv & imask));
                }
                const int64_t qrow = (int64_t)h * N + r0 + 32 * quad + r;
                float es = -INFINITY;
                int ei = 0x7fffffff;
                if (cand >= 0) {
                    es = exact_score_g<D>(Q + qrow * D, cent + (hk * n_blocks + cand) * (int64_t)D);
                    ei = cand;
                }
                int rank = 0;
#pragma unroll
                for (int src = 0; src < LS; ++src) {
                    const float os = __shfl_sync(0xffffffffu, es, src);
                    const int oi = __shfl_sync(0xffffffffu, ei, src);
                    rank += better(os, oi, es, ei) ? 1 : 0;
                }
                uint32_t sel = __ballot_sync(0xffffffffu, cand >= 0 && rank < top_k);
#pragma unroll
                for (int p = 0; p < KMAX; ++p) {
                    const int l = sel != 0u ? __ffs(sel) - 1 : 0;
                    sel &= sel - 1u;
                    const int v = __shfl_sync(0xffffffffu, ei, l);
                    if (lane == r && p < top_k) res[p] = v;
                }
            }
            if (status == 2) {
                // queued twice: as a row (recheck[0] counts, rows after the
                // tile flags) and, by its tile's first such row, as a tile
                // (recheck[1] counts, ids from recheck[2]); the pass that
                // runs picks whichever is cheaper (route_recheck_kernel /
                // route_topk_fp32_kernel tile-list mode)
                const int tile_id = h * n_tiles + t;
                if (atomicExch(recheck + 2 + bh * n_tiles + tile_id, 1) == 0) {
                    const int slot = atomicAdd(recheck + 1, 1);
                    recheck[2 + slot] = tile_id;
                }
                const int rslot = atomicAdd(recheck, 1);
                recheck[2 + 2 * bh * n_tiles + rslot] = (int)((int64_t)h * N + my_i);
            }
            if (valid) write_row<KMAX>(topk + ((int64_t)h * N + my_i) * width, res, top_k, own, width);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// Queued rows, one warp per row: every candidate j < own scored with the fp32
// chain (lanes stride over j, so each lane sees its candidates in ascending
// order), per-lane top-k lists, then a k-round warp merge by (score desc,
// index asc). Bitwise the fp32 router's selection for the row.
template <int D, int KMAX>
__global__ void __launch_bounds__(256)
route_recheck_kernel(const __nv_bfloat16* __restrict__ Q, const float* __restrict__ cent, int64_t N, int B,
                     int top_k, int kv_group, const int* __restrict__ recheck, int n_tiles_all,
                     int32_t* __restrict__ topk) {
    const int lane = threadIdx.x & 31;
    const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nw = (int)((gridDim.x * blockDim.x) >> 5);
    const int n_blocks = (int)((N + B - 1) / B);
    const int width = top_k + 1;
    // rows only while they are few per listed tile (about 16); otherwise the
    // tile pass re-routes whole tiles
    const int count = recheck[0] <= 16 * recheck[1] ? recheck[0] : 0;
    const int* rows = recheck + 2 + 2 * n_tiles_all;
    for (int r = gw; r < count; r += nw) {
        const int64_t row = rows[r];
        const int64_t h = row / N, i = row - h * N;
        const int own = (int)(i / B);
        const float* Ch = cent + (h / kv_group) * (int64_t)n_blocks * D;
        float qv[D];
#pragma unroll
        for (int dd = 0; dd < D; dd += 8) {
            float x[8];
            ld8f(Q + row * D + dd, x);
#pragma unroll
            for (int e = 0; e < 8; ++e) qv[dd + e] = x[e];
        }
        float ts[KMAX];
        int ti[KMAX];
#pragma unroll
        for (int u = 0; u < KMAX; ++u) {
            ts[u] = -INFINITY;
            ti[u] = 0x7fffffff;
        }
        for (int j = lane; j < own; j += 32) list_insert<KMAX>(ts, ti, exact_score<D>(qv, Ch + (int64_t)j * D), j);
        int res[KMAX];
        int head = 0;
        for (int p = 0; p < KMAX; ++p) {
            float s = -INFINITY;
            int ix = 0x7fffffff;
#pragma unroll
            for (int u = 0; u < KMAX; ++u)
                if (u == head) {
                    s = ts[u];
                    ix = ti[u];
                }
            float bs = s;
            int bi = ix;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float os = __shfl_xor_sync(0xffffffffu, bs, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (better(os, oi, bs, bi)) {
                    bs = os;
                    bi = oi;
                }
            }
            res[p] = bi;
            if (bi == ix && bi != 0x7fffffff) ++head;
        }
        if (lane == 0) write_row<KMAX>(topk + row * width, res, top_k, own, width);
    }
}

// centroids fp32 [rows, D] -> bf16 hi / lo split terms [2][rows][D] and the
// per-(K/V head) max squared centroid norm (for the guard); one warp per row
__global__ void centroid_split2_kernel(const float* __restrict__ cent, int64_t rows, int D, int n_blocks,
                                       __nv_bfloat16* __restrict__ split, float* __restrict__ cmax2) {
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    float n2 = 0.f;
    for (int c = lane; c < D; c += 32) {
        const float v = cent[r * D + c];
        const __nv_bfloat16 hi = __float2bfloat16(v);
        const __nv_bfloat16 lo = __float2bfloat16(v - __bfloat162float(hi));
        split[r * D + c] = hi;
        split[rows * D + r * D + c] = lo;
        n2 = fmaf(v, v, n2);
    }
    n2 = warp_sum(n2);
    if (lane == 0) atomicMax(reinterpret_cast<int*>(cmax2) + r / n_blocks, __float_as_int(n2));
}

}  // namespace rtc

bool make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint32_t cols, uint32_t box_rows);
template <int D, int KMAX>
int launch_route_fp32_tiles(const void* q, const float* cent, int64_t bh, int kv_group, int64_t N, int B, int top_k,
                            int32_t* topk, const int* tiles, const int* rows_count, cudaStream_t s);

// workspace: [split bf16 2 x rows x D][cmax2 f32 x bh_kv]
//            [row count, tile count, bh * n_tiles tile ids, bh * n_tiles flags, bh * N rows]
size_t route_tc_ws_bytes(int64_t bh, int64_t N, int B) {
    const int64_t n = ceil_div(N, B);
    return align_up((size_t)2 * bh * n * 128 * 2, 256) + align_up((size_t)bh * 4, 256) +
           align_up((size_t)(2 + 2 * bh * ceil_div(N, 128) + bh * N) * 4, 256);
}

template <int D, int KMAX>
int launch_route_tc(const void* q, const float* cent, int64_t bh, int kv_group, int64_t N, int B, int top_k,
                    int32_t* topk, void* ws, cudaStream_t s) {
    using namespace rtc;
    const int64_t n = ceil_div(N, B);
    const int64_t bh_kv = bh / kv_group;
    const int64_t rows = bh_kv * n;
    uint8_t* w = (uint8_t*)ws;
    __nv_bfloat16* split = (__nv_bfloat16*)w;
    w += align_up((size_t)2 * bh * n * 128 * 2, 256);
    float* cmax2 = (float*)w;
    w += align_up((size_t)bh * 4, 256);
    int* recheck = (int*)w;
    cudaMemsetAsync(cmax2, 0, (size_t)bh_kv * 4, s);
    const int n_tiles = (int)ceil_div(N, kM);
    cudaMemsetAsync(recheck, 0, (size_t)(2 + 2 * bh * n_tiles) * 4, s);
    centroid_split2_kernel<<<(unsigned)ceil_div(rows * 32, 256), 256, 0, s>>>(cent, rows, D, (int)n, split, cmax2);
    int st = check_launch("centroid_split2_kernel");
    if (st) return st;
    CUtensorMap tm_q, tm_c;
    if (!make_tmap_bf16(&tm_q, q, (uint64_t)(bh * N), D, kM) ||
        !make_tmap_bf16(&tm_c, split, (uint64_t)(2 * rows), D, kN))
        return MOBA_ERR_CUDA;
    int idx_bits = 1;
    while ((1ll << idx_bits) < n) ++idx_bits;
    if (idx_bits > 20) return MOBA_ERR_UNSUPPORTED;
    auto go = [&](auto tt_tag, auto lx_tag) -> int {
        constexpr int TT = decltype(tt_tag)::value;
        constexpr int LX = decltype(lx_tag)::value;
        using G = Geo<D, TT>;
        const int n_groups = (int)ceil_div(n_tiles, G::T);
        const int64_t units = bh * n_groups;
        if (units >= (1ll << 31)) return MOBA_ERR_UNSUPPORTED;
        auto kern = route_tc_kernel<D, KMAX, TT, LX>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::kSmem);
        const unsigned grid = (unsigned)std::min<int64_t>(units, kNumSMs);
        kern<<<grid, G::kThreads, G::kSmem, s>>>(tm_q, tm_c, (const __nv_bfloat16*)q, cent, cmax2, N, B, top_k, rows,
                                                 kv_group, (int)bh, n_tiles, n_groups, idx_bits, topk, recheck);
        return check_launch("route_tc_kernel");
    };
    // d = 64: units of 4 query tiles (21 warps); per-row lists of k + 2 keys,
    // k + 3 from 256K tokens. Measured route+varlen, 32 heads d64 (tc plans
    // bitwise the fp32 router's in every variant):
    //            3 tiles, k+4 | 3 tiles, k+2 | 4 tiles, k+3 | 4 tiles, k+2
    //   64K       0.926 ms    |   0.897      |   0.876      |   0.860
    //   128K        -         |   2.26       |   2.22       |   2.17
    //   256K        -         |   6.51       |   6.11       |   6.20
    //   512K      19.16 (4 tiles)  -        |  18.71       |  22.5
    // d = 128: units of 2 tiles, k + 2 (64K 0.952 -> 0.908 ms vs k + 4)
    using I2 = std::integral_constant<int, 2>;
    using I3 = std::integral_constant<int, 3>;
    using I4 = std::integral_constant<int, 4>;
    if constexpr (D == 64)
        st = (N >= (1 << 18)) ? go(I4{}, I3{}) : go(I4{}, I2{});
    else
        st = go(I2{}, I2{});
    if (st) return st;
    route_recheck_kernel<D, KMAX><<<kNumSMs * 2, 256, 0, s>>>((const __nv_bfloat16*)q, cent, N, B, top_k, kv_group,
                                                              recheck, (int)(bh * n_tiles), topk);
    st = check_launch("route_recheck_kernel");
    if (st) return st;
    return launch_route_fp32_tiles<D, KMAX>(q, cent, bh, kv_group, N, B, top_k, topk, recheck + 1, recheck, s);
}

#define MOBA_RTC_INST(D, K)                                                                                  \
    template int launch_route_tc<D, K>(const void*, const float*, int64_t, int, int64_t, int, int, int32_t*, \
                                       void*, cudaStream_t);
MOBA_RTC_INST(64, 1)
MOBA_RTC_INST(64, 2)
MOBA_RTC_INST(64, 4)
MOBA_RTC_INST(64, 8)
MOBA_RTC_INST(64, 16)
MOBA_RTC_INST(64, 32)
MOBA_RTC_INST(128, 1)
MOBA_RTC_INST(128, 2)
MOBA_RTC_INST(128, 4)
MOBA_RTC_INST(128, 8)
MOBA_RTC_INST(128, 16)
MOBA_RTC_INST(128, 32)
#undef MOBA_RTC_INST

}  // namespace moba
