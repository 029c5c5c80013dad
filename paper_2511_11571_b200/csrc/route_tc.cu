// Tensor-core top-k routing with an exactness guard (select_topk,
// src/router.py:49-120, tensor-core mode).
//
// Scores S = Q (C_hi + C_lo)^T on tcgen05: the fp32 centroids are split into
// two bf16 terms (|c - c_hi - c_lo| <= 2^-16 |c|), Q is bf16 (exact), fp32
// accumulation in TMEM. A CTA owns a tile of 128 queries (TMEM lanes) and
// streams 128-centroid chunks (MMA N = 128) through a double-buffered TMEM
// accumulator; tiles are launched longest first (the last tiles of a head
// see the most past blocks).
//
// Warps (288 threads):
//   0      TMA (Q tile once, centroid chunks through CS smem stages) and MMA
//          issue, one elected lane
//   1-8    selection: the two warps of a TMEM lane quadrant split each chunk
//          (columns 0-63 / 64-127). Per 16 candidates a thread builds a
//          bitmask of the scores above its running threshold (two
//          instructions per candidate); only when some lane has a hit are
//          the 16 scores staged in shared memory and inserted, in ascending
//          block order, into a sorted list of LS = top_k + 2 (ties keep the
//          lower block index first, src/router.py:95-98).
//
// Exactness: the list keeps the two best candidates beyond the top k, so the
// tensor-core selection can be certified against the fp32 router
// (route_topk_fp32_kernel, whose scores are the fp32 FFMA chain over d):
//   eps(row) = kEps(D) * |q| * max_j |c_j| bounds |s_tc - s_fp32| for every
//   candidate of the row (split error 2^-16, tensor-core accumulation and
//   the FFMA chain, x2 margin);
//   s_k - s_{k+1} > 2 eps  -> the tensor-core top k IS the fp32 top k;
//   s_k - s_{k+2} > 2 eps  -> the fp32 top k lies inside the k + 2 listed
//                             candidates: they are rescored with the fp32
//                             FFMA chain and reselected exactly (in-kernel);
//   otherwise               -> the row is queued and route_recheck_kernel
//                             reselects it over all its candidates in fp32.
// The output is therefore bitwise the fp32 router's (the parity mode) for
// every row.
#include "common.cuh"
#include "sm100.cuh"

namespace moba {
namespace rtc {

constexpr int kM = 128;            // queries per tile (TMEM lanes)
constexpr int kN = 128;            // centroids per chunk (MMA N)
constexpr int kSplits = 2;         // bf16 hi + lo terms of the fp32 centroids
constexpr int kSelWarps = 8;
constexpr int kThreads = 32 * (1 + kSelWarps);
constexpr int kGrp = 16;           // candidates per filter group
constexpr int kStgStride = kGrp + 4;   // floats per lane in the staging area (conflict-free STS.128)

template <int D>
struct Geo {
    static constexpr int CS = (D == 64) ? 2 : 1;                      // centroid smem stages
    static constexpr uint32_t kQ = kM * D * 2;
    static constexpr uint32_t kCterm = kN * D * 2;
    static constexpr uint32_t kC = kSplits * kCterm;
    static constexpr uint32_t kStg = kSelWarps * 32 * kStgStride * 4;
    static constexpr uint32_t kBars = 128;
    static constexpr uint32_t kSmem = 1024 + kQ + CS * kC + kStg + kBars;
    // |s_tc - s_fp32| <= kEps * |q| * max|c|, with
    //   split:       2^-16 (two bf16 terms)
    //   tc accum.:   2 * (kSplits * D / 16 + 1) * 2^-23 (per K=16 MMA step, truncating)
    //   fp32 chain:  D * 2^-24 (sequential FFMA over d)
    // and a 2x safety margin
    static constexpr float kEps = 2.0f * (1.52587890625e-05f + 2.0f * (kSplits * D / 16 + 1) * 1.1920928955078125e-07f +
                                          D * 5.9604644775390625e-08f);
};

struct Bars {
    uint64_t c_full[2], c_empty[2], s_full[2], s_free[2];
    uint32_t tmem;
};

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

// exact fp32 score = the fp32 router's FFMA chain (dd = 0 .. D-1 from 0),
// q row from the bf16 SW128 smem tile (row `row` of a 128-row tile)
template <int D>
MOBA_DEV float exact_score_smem(uint32_t sq, int row, const float* __restrict__ c) {
    float acc = 0.f;
#pragma unroll
    for (int cg = 0; cg < D / 8; ++cg) {
        const int sl = cg >> 3, ch = cg & 7;
        const int4 raw = lds128i(sq + sl * 128 * 128 + row * 128 + ((ch ^ (row & 7)) << 4));
        const uint32_t u4[4] = {(uint32_t)raw.x, (uint32_t)raw.y, (uint32_t)raw.z, (uint32_t)raw.w};
        const float4 v0 = __ldg(reinterpret_cast<const float4*>(c + cg * 8));
        const float4 v1 = __ldg(reinterpret_cast<const float4*>(c + cg * 8) + 1);
        const float cv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 f = unpack_bf16(u4[e]);
            acc = fmaf(f.x, cv[2 * e], acc);
            acc = fmaf(f.y, cv[2 * e + 1], acc);
        }
    }
    return acc;
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

template <int D, int KMAX>
__global__ void __launch_bounds__(kThreads, 2)
route_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_c,
                const __nv_bfloat16* __restrict__ Q, const float* __restrict__ cent, const float* __restrict__ cmax2,
                int64_t N, int B, int top_k, int64_t split_rows, int kv_group, int n_tiles,
                int32_t* __restrict__ topk, int* __restrict__ recheck) {
    using namespace sm100;
    using G = Geo<D>;
    constexpr int LS = KMAX + 2;
    constexpr int SL = D / 64;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sq = smem_u32(smem);
    const uint32_t sc = sq + G::kQ;
    float* stg = reinterpret_cast<float*>(smem + G::kQ + G::CS * G::kC);
    Bars* bars = reinterpret_cast<Bars*>(smem + G::kQ + G::CS * G::kC + G::kStg);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t h = blockIdx.x;
    const int tile = n_tiles - 1 - (int)blockIdx.y;          // longest tiles first
    const int64_t r0 = (int64_t)tile * kM;
    const int n_blocks = (int)((N + B - 1) / B);
    const int width = top_k + 1;
    const int max_own = (int)((min64(r0 + kM, N) - 1) / B);
    const int n_chunks = (max_own + kN - 1) / kN;
    const int64_t hk = h / kv_group;

    if (warp == 0) tmem_alloc(&bars->tmem, 2 * kN);
    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->c_full[i], 1);
            mbar_init(&bars->c_empty[i], 1);
            mbar_init(&bars->s_full[i], 1);
            mbar_init(&bars->s_free[i], kSelWarps);
        }
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA + MMA
        if (n_chunks > 0) {
            const uint32_t idesc = idesc_bf16(kM, kN, false, false);
            auto load = [&](int c) {
                const int st = c % G::CS;
                const uint32_t dst = sc + st * G::kC;
                if (lane == 0) {
                    mbar_expect_tx(&bars->c_full[st], G::kC + (c == 0 ? G::kQ : 0));
                    if (c == 0)
#pragma unroll
                        for (int sl = 0; sl < SL; ++sl)
                            tma_load_2d(sq + sl * kM * 128, &tm_q, sl * 64, (int)(h * N + r0), &bars->c_full[st]);
#pragma unroll
                    for (int t = 0; t < kSplits; ++t)
#pragma unroll
                        for (int sl = 0; sl < SL; ++sl)
                            tma_load_2d(dst + t * G::kCterm + sl * kN * 128, &tm_c, sl * 64,
                                        (int)(t * split_rows + hk * n_blocks + (int64_t)c * kN), &bars->c_full[st]);
                }
                __syncwarp();
            };
            for (int c = 0; c < min(G::CS, n_chunks); ++c) load(c);
            for (int c = 0; c < n_chunks; ++c) {
                const int st = c % G::CS, slot = c & 1;
                mbar_wait(&bars->c_full[st], (c / G::CS) & 1);
                if (c >= 2) mbar_wait(&bars->s_free[slot], ((c >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t cb = sc + st * G::kC;
#pragma unroll
                for (int t = 0; t < kSplits; ++t)
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const int sl = kk >> 2, ke = (kk & 3) * 16;
                        umma_bf16_w(tmem + slot * kN, desc_kmajor(sq + sl * kM * 128, ke),
                                    desc_kmajor(cb + t * G::kCterm + sl * kN * 128, ke), idesc, t > 0 || kk > 0);
                    }
                umma_commit_w(&bars->s_full[slot]);
                umma_commit_w(&bars->c_empty[st]);
                if (c + G::CS < n_chunks) {
                    mbar_wait(&bars->c_empty[st], (c / G::CS) & 1);   // MMA(c) has read the stage
                    load(c + G::CS);
                }
            }
        }
    } else {
        // ------------------------------------------------------------ selection
        const int sw = warp - 1;
        const int quad = warp & 3, half = sw >> 2;
        const int row = 32 * quad + lane;
        const int64_t my_i = r0 + row;
        const bool valid = my_i < N;
        const int my_own = (int)(min64(my_i, N - 1) / B);
        const uint32_t lane_off = (uint32_t)(32 * quad) << 16;
        float* my_stg = stg + (sw * 32 + lane) * kStgStride;
        float ts[LS];
        int ti[LS];
#pragma unroll
        for (int u = 0; u < LS; ++u) {
            ts[u] = -INFINITY;
            ti[u] = 0x7fffffff;
        }
        for (int c = 0; c < n_chunks; ++c) {
            const int slot = c & 1;
            const int j0 = c * kN + 64 * half;
            const int lim = valid ? max(0, min(64, my_own - j0)) : 0;   // strictly-past blocks only
            mbar_wait(&bars->s_full[slot], (c >> 1) & 1);
            tc_fence_after();
            float sv[64];
            if (__any_sync(0xffffffffu, lim > 0)) {
                tmem_ld32(tmem + slot * kN + 64 * half + lane_off, *reinterpret_cast<float(*)[32]>(&sv[0]));
                tmem_ld32(tmem + slot * kN + 64 * half + 32 + lane_off, *reinterpret_cast<float(*)[32]>(&sv[32]));
                tmem_ld_wait();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->s_free[slot]);
            if (!__any_sync(0xffffffffu, lim > 0)) continue;
#pragma unroll
            for (int g = 0; g < 64 / kGrp; ++g) {
                const float thr = ts[LS - 1];
                uint32_t m = 0;
#pragma unroll
                for (int i = 0; i < kGrp; ++i) m |= (sv[g * kGrp + i] > thr) ? (1u << i) : 0u;
                const int rem = lim - g * kGrp;
                m &= rem >= kGrp ? 0xffffu : (rem > 0 ? (1u << rem) - 1u : 0u);
                if (!__any_sync(0xffffffffu, m != 0)) continue;
                if (m != 0) {
#pragma unroll
                    for (int i = 0; i < kGrp; i += 4)
                        *reinterpret_cast<float4*>(my_stg + i) =
                            make_float4(sv[g * kGrp + i], sv[g * kGrp + i + 1], sv[g * kGrp + i + 2], sv[g * kGrp + i + 3]);
                }
                while (__any_sync(0xffffffffu, m != 0)) {
                    float s = -INFINITY;
                    int j = 0x7fffffff;
                    if (m != 0) {
                        const int b = __ffs(m) - 1;
                        m &= m - 1;
                        s = my_stg[b];
                        j = j0 + g * kGrp + b;
                    }
                    list_insert<LS>(ts, ti, s > ts[LS - 1] ? s : -INFINITY, j);
                }
            }
        }
        // ---- merge the two halves' lists (the C stages are free now)
        float* ms = reinterpret_cast<float*>(smem + G::kQ);            // [LS][128]
        int* mi = reinterpret_cast<int*>(smem + G::kQ + LS * kM * 4);  // [LS][128]
        if (half == 1) {
#pragma unroll
            for (int u = 0; u < LS; ++u) {
                ms[u * kM + row] = ts[u];
                mi[u * kM + row] = ti[u];
            }
        }
        named_bar(1 + quad, 64);
        if (half == 0 && valid) {
            float rs[LS];
            int ri[LS];
            {
                int a = 0, b = 0;
                float bsc = ms[row];
                int bix = mi[row];
#pragma unroll
                for (int u = 0; u < LS; ++u) {
                    float asc = -INFINITY;
                    int aix = 0x7fffffff;
#pragma unroll
                    for (int v = 0; v < LS; ++v)
                        if (v == a) {
                            asc = ts[v];
                            aix = ti[v];
                        }
                    const bool take_a = better(asc, aix, bsc, bix);
                    rs[u] = take_a ? asc : bsc;
                    ri[u] = take_a ? aix : bix;
                    if (take_a) {
                        ++a;
                    } else {
                        ++b;
                        bsc = (b < LS) ? ms[b * kM + row] : -INFINITY;
                        bix = (b < LS) ? mi[b * kM + row] : 0x7fffffff;
                    }
                }
            }
            int res[KMAX];
#pragma unroll
            for (int u = 0; u < KMAX; ++u) res[u] = ri[u];
            if (my_own > top_k) {
                // ---- exactness guard
                float sk = -INFINITY, sk1 = -INFINITY, sk2 = -INFINITY;
#pragma unroll
                for (int u = 0; u < LS; ++u) {
                    if (u == top_k - 1) sk = rs[u];
                    if (u == top_k) sk1 = rs[u];
                    if (u == top_k + 1) sk2 = rs[u];
                }
                float qn = 0.f;
#pragma unroll
                for (int cg = 0; cg < D / 8; ++cg) {
                    const int sl = cg >> 3, ch = cg & 7;
                    const int4 raw = lds128i(sq + sl * kM * 128 + row * 128 + ((ch ^ (row & 7)) << 4));
                    const uint32_t u4[4] = {(uint32_t)raw.x, (uint32_t)raw.y, (uint32_t)raw.z, (uint32_t)raw.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 f = unpack_bf16(u4[e]);
                        qn = fmaf(f.x, f.x, fmaf(f.y, f.y, qn));
                    }
                }
                const float eps = G::kEps * sqrtf(qn) * sqrtf(__ldg(cmax2 + hk));
                if (!(sk - sk1 > 2.f * eps)) {
                    if (sk - sk2 > 2.f * eps) {
                        // the fp32 top k lies among the k + 2 listed candidates:
                        // rescore them with the fp32 chain and reselect exactly
                        const float* Ch = cent + hk * (int64_t)n_blocks * D;
                        float es[KMAX + 2];
                        int ei[KMAX + 2];
#pragma unroll
                        for (int u = 0; u < KMAX + 2; ++u) {
                            ei[u] = (u < top_k + 2) ? ri[u] : 0x7fffffff;
                            es[u] = (ei[u] != 0x7fffffff) ? exact_score_smem<D>(sq, row, Ch + (int64_t)ei[u] * D) : -INFINITY;
                        }
                        // selection sort of the top_k by (score desc, index asc)
#pragma unroll
                        for (int p = 0; p < KMAX; ++p) {
#pragma unroll
                            for (int u = p + 1; u < KMAX + 2; ++u) {
                                if (better(es[u], ei[u], es[p], ei[p])) {
                                    const float t = es[p];
                                    es[p] = es[u];
                                    es[u] = t;
                                    const int ti2 = ei[p];
                                    ei[p] = ei[u];
                                    ei[u] = ti2;
                                }
                            }
                            res[p] = ei[p];
                        }
                    } else {
                        // two near-ties at the boundary: full fp32 reselection of the row
                        const int slotq = atomicAdd(recheck, 1);
                        recheck[1 + slotq] = (int)(h * N + my_i);
                    }
                }
            }
            write_row<KMAX>(topk + (h * N + my_i) * width, res, top_k, my_own, width);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 2 * kN);
    }
}

// One warp per queued row: every candidate j < own scored with the fp32
// chain (lanes stride over j, so each lane sees its candidates in ascending
// order), per-lane top-k lists, then a k-round warp merge by (score desc,
// index asc). Bitwise the fp32 router's selection for the row.
template <int D, int KMAX>
__global__ void __launch_bounds__(256)
route_recheck_kernel(const __nv_bfloat16* __restrict__ Q, const float* __restrict__ cent, int64_t N, int B,
                     int top_k, int kv_group, const int* __restrict__ recheck, int32_t* __restrict__ topk) {
    const int lane = threadIdx.x & 31;
    const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nw = (int)((gridDim.x * blockDim.x) >> 5);
    const int n_blocks = (int)((N + B - 1) / B);
    const int width = top_k + 1;
    const int count = *recheck;
    for (int r = gw; r < count; r += nw) {
        const int64_t row = recheck[1 + r];
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

// workspace: [split bf16 2 x rows x D][cmax2 f32 x bh_kv][recheck int (1 + bh * N)]
size_t route_tc_ws_bytes(int64_t bh, int64_t N, int B) {
    const int64_t n = ceil_div(N, B);
    return align_up((size_t)2 * bh * n * 128 * 2, 256) + align_up((size_t)bh * 4, 256) +
           align_up((size_t)(1 + bh * N) * 4, 256);
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
    cudaMemsetAsync(recheck, 0, 4, s);
    centroid_split2_kernel<<<(unsigned)ceil_div(rows * 32, 256), 256, 0, s>>>(cent, rows, D, (int)n, split, cmax2);
    int st = check_launch("centroid_split2_kernel");
    if (st) return st;
    CUtensorMap tm_q, tm_c;
    if (!make_tmap_bf16(&tm_q, q, (uint64_t)(bh * N), D, kM) ||
        !make_tmap_bf16(&tm_c, split, (uint64_t)(2 * rows), D, kN))
        return MOBA_ERR_CUDA;
    const int n_tiles = (int)ceil_div(N, kM);
    auto kern = route_tc_kernel<D, KMAX>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Geo<D>::kSmem);
    kern<<<dim3((unsigned)bh, (unsigned)n_tiles), kThreads, Geo<D>::kSmem, s>>>(
        tm_q, tm_c, (const __nv_bfloat16*)q, cent, cmax2, N, B, top_k, rows, kv_group, n_tiles, topk, recheck);
    st = check_launch("route_tc_kernel");
    if (st) return st;
    route_recheck_kernel<D, KMAX><<<kNumSMs * 2, 256, 0, s>>>((const __nv_bfloat16*)q, cent, N, B, top_k, kv_group,
                                                              recheck, topk);
    return check_launch("route_recheck_kernel");
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
