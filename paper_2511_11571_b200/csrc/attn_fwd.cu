// Forward: gather-and-densify over key blocks (moba_forward,
// src/attention.py:147-182; paper Alg. 1), key-block-major.
//
// Work item = (head, key block j, 64-row tile of block j's varlen slice).
// The CTA gathers the tile's query rows (flat_queries) into shared memory,
// streams K_j / V_j, and runs S = Q K_j^T, the token-causal mask
// (src/attention.py:127-133), an online softmax over 64-key chunks
// (SoftmaxState.update, src/attention.py:60-68) and P V_j on the tensor
// cores. Each (query, block) pair yields one partial (O_s normalised, bf16;
// lse_s fp32) stored at its flat position; moba_combine merges a query's
// partials into O and LSE (SoftmaxState.finalize, src/attention.py:70-74).
//
// This is the legacy-MMA (mma.sync m16n8k16) path.
#include "common.cuh"
#include "sm100.cuh"
#include <cstdlib>

namespace moba {

constexpr int kFwdBM = 64;        // gathered query rows per item
constexpr int kFwdThreads = 128;  // 4 warps x 16 rows
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

struct FwdItem {
    int32_t hj;    // head * n_blocks + j
    int32_t row0;  // first slice row of the tile
};

template <int D>
struct FwdSmem {
    static constexpr int RB = D * 2;  // bytes per bf16 row
};

// Q rows of the tile; K_j, V_j padded to BP rows (multiple of 64), zero filled.
template <int D>
__global__ void __launch_bounds__(kFwdThreads)
moba_fwd_mma_kernel(const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ K,
                    const __nv_bfloat16* __restrict__ V, int64_t N, int B, int BP, int width,
                    const int32_t* __restrict__ counts, const int32_t* __restrict__ offsets,
                    const int32_t* __restrict__ flat, const FwdItem* __restrict__ items,
                    const int32_t* __restrict__ n_items_ptr, float scale_log2,
                    __nv_bfloat16* __restrict__ part_o, float* __restrict__ part_lse) {
    constexpr int RB = D * 2;
    constexpr int CH = D / 8;  // 16-byte chunks per row
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* q_s = smem;
    uint8_t* k_s = q_s + kFwdBM * RB;
    uint8_t* v_s = k_s + BP * RB;
    int32_t* qid_s = reinterpret_cast<int32_t*>(v_s + BP * RB);

    const int n_blocks = (int)((N + B - 1) / B);
    const int n_items = *n_items_ptr;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, t4 = lane & 3;

    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const FwdItem item = items[it];
        const int64_t h = item.hj / n_blocks;
        const int j = item.hj % n_blocks;
        const int cnt = counts[item.hj];
        const int rows = min(kFwdBM, cnt - item.row0);
        const int64_t pbase = (int64_t)offsets[item.hj] + item.row0;  // head-local flat position
        const int32_t* fl = flat + h * N * width + pbase;
        const int64_t k0 = (int64_t)j * B;
        const int klen = (int)min64(B, N - k0);
        const __nv_bfloat16* Qh = Q + h * N * D;
        const __nv_bfloat16* Kh = K + (h * N + k0) * D;
        const __nv_bfloat16* Vh = V + (h * N + k0) * D;

        __syncthreads();  // previous item's smem readers are done
        if (tid < kFwdBM) qid_s[tid] = (tid < rows) ? fl[tid] : -1;
        __syncthreads();
        // gather Q rows (zero fill past the tile)
        for (int e = tid; e < kFwdBM * CH; e += kFwdThreads) {
            int r = e / CH, c = e % CH;
            int qi = qid_s[r];
            cp_async16(smem_u32(q_s + swz<RB>(r, c)), Qh + (int64_t)max(qi, 0) * D + c * 8, qi >= 0);
        }
        // K_j, V_j (zero fill past the block / sequence end)
        for (int e = tid; e < BP * CH; e += kFwdThreads) {
            int r = e / CH, c = e % CH;
            bool ok = r < klen;
            int rr = ok ? r : 0;
            cp_async16(smem_u32(k_s + swz<RB>(r, c)), Kh + (int64_t)rr * D + c * 8, ok);
            cp_async16(smem_u32(v_s + swz<RB>(r, c)), Vh + (int64_t)rr * D + c * 8, ok);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();

        const int m0 = warp * 16;
        const int q_lo = qid_s[m0 + g];
        const int q_hi = qid_s[m0 + g + 8];
        // Q fragments for the whole d range
        uint32_t qa[D / 16][4];
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
            int r = m0 + (lane & 7) + ((lane >> 3) & 1) * 8;
            int c = kk * 2 + (lane >> 4);
            ldmatrix_x4(smem_u32(q_s + swz<RB>(r, c)), qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
        }
        float o[D / 8][4];
#pragma unroll
        for (int nt = 0; nt < D / 8; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
        float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;

        for (int kc = 0; kc < BP; kc += 64) {
            float s[8][4];
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
                for (int np = 0; np < 4; ++np) {  // pairs of n-tiles (16 keys)
                    int key = kc + np * 16 + (lane & 7) + (lane >> 4) * 8;
                    int c = kk * 2 + ((lane >> 3) & 1);
                    uint32_t b0, b1, b2, b3;
                    ldmatrix_x4(smem_u32(k_s + swz<RB>(key, c)), b0, b1, b2, b3);
                    mma_bf16_16816(s[2 * np], qa[kk], b0, b1);
                    mma_bf16_16816(s[2 * np + 1], qa[kk], b2, b3);
                }
            }
            // scale into the log2 domain and mask: key col c valid iff
            // c < klen and k0 + c <= query
            float cm_lo = -INFINITY, cm_hi = -INFINITY;
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    int col = kc + nt * 8 + 2 * t4 + (e & 1);
                    int qq = (e < 2) ? q_lo : q_hi;
                    bool ok = col < klen && (k0 + col) <= (int64_t)qq;
                    float v = ok ? s[nt][e] * scale_log2 : -INFINITY;
                    s[nt][e] = v;
                    if (e < 2) cm_lo = fmaxf(cm_lo, v); else cm_hi = fmaxf(cm_hi, v);
                }
            }
            cm_lo = fmaxf(cm_lo, __shfl_xor_sync(0xffffffffu, cm_lo, 1));
            cm_lo = fmaxf(cm_lo, __shfl_xor_sync(0xffffffffu, cm_lo, 2));
            cm_hi = fmaxf(cm_hi, __shfl_xor_sync(0xffffffffu, cm_hi, 1));
            cm_hi = fmaxf(cm_hi, __shfl_xor_sync(0xffffffffu, cm_hi, 2));
            float mn_lo = fmaxf(m_lo, cm_lo), mn_hi = fmaxf(m_hi, cm_hi);
            // rows with no visible key yet keep a finite reference point
            float ref_lo = (mn_lo == -INFINITY) ? 0.f : mn_lo;
            float ref_hi = (mn_hi == -INFINITY) ? 0.f : mn_hi;
            float al_lo = fast_exp2(m_lo - ref_lo), al_hi = fast_exp2(m_hi - ref_hi);
            m_lo = mn_lo;
            m_hi = mn_hi;
            l_lo *= al_lo;
            l_hi *= al_hi;
#pragma unroll
            for (int nt = 0; nt < D / 8; ++nt) {
                o[nt][0] *= al_lo;
                o[nt][1] *= al_lo;
                o[nt][2] *= al_hi;
                o[nt][3] *= al_hi;
            }
            uint32_t pa[4][4];  // P as A fragments, 4 k16 slices
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
                float p0 = fast_exp2(s[nt][0] - ref_lo);
                float p1 = fast_exp2(s[nt][1] - ref_lo);
                float p2 = fast_exp2(s[nt][2] - ref_hi);
                float p3 = fast_exp2(s[nt][3] - ref_hi);
                l_lo += p0 + p1;
                l_hi += p2 + p3;
                pa[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16(p0, p1);
                pa[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16(p2, p3);
            }
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
                for (int np = 0; np < D / 16; ++np) {
                    int key = kc + ks * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
                    int c = np * 2 + (lane >> 4);
                    uint32_t b0, b1, b2, b3;
                    ldmatrix_x4_trans(smem_u32(v_s + swz<RB>(key, c)), b0, b1, b2, b3);
                    mma_bf16_16816(o[2 * np], pa[ks], b0, b1);
                    mma_bf16_16816(o[2 * np + 1], pa[ks], b2, b3);
                }
            }
        }
        l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 1);
        l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 2);
        l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 1);
        l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 2);
        const float inv_lo = 1.f / l_lo, inv_hi = 1.f / l_hi;
        __nv_bfloat16* po = part_o + (h * N * width + pbase) * D;
        float* pl = part_lse + h * N * width + pbase;
        const int r_lo = m0 + g, r_hi = m0 + g + 8;
#pragma unroll
        for (int nt = 0; nt < D / 8; ++nt) {
            int col = nt * 8 + 2 * t4;
            if (r_lo < rows)
                *reinterpret_cast<uint32_t*>(po + (int64_t)r_lo * D + col) =
                    pack_bf16(o[nt][0] * inv_lo, o[nt][1] * inv_lo);
            if (r_hi < rows)
                *reinterpret_cast<uint32_t*>(po + (int64_t)r_hi * D + col) =
                    pack_bf16(o[nt][2] * inv_hi, o[nt][3] * inv_hi);
        }
        if (t4 == 0) {
            if (r_lo < rows) pl[r_lo] = (m_lo + __log2f(l_lo)) * kLn2;
            if (r_hi < rows) pl[r_hi] = (m_hi + __log2f(l_hi)) * kLn2;
        }
    }
}


// ---------------------------------------------------------------- tcgen05 path
// One CTA (4 warps, one gathered query row per thread) per item at a time,
// items in a contiguous per-CTA range so consecutive items usually share
// (head, block) and K_j / V_j stay resident in shared memory.
//   S[128 x BP] = Q_g K_j^T      (tcgen05.mma, fp32 in TMEM cols [0, BP))
//   softmax rows from TMEM (tcgen05.ld), P -> smem (bf16, SW128 K-major)
//   O[128 x D]  = P V_j          (tcgen05.mma, V as MN-major B operand)
constexpr int kTcM = 128;

template <int D>
__global__ void __launch_bounds__(128, 1)
moba_fwd_tc_kernel(const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ K,
                   const __nv_bfloat16* __restrict__ V, int64_t N, int B, int BP, int width,
                   const int32_t* __restrict__ counts, const int32_t* __restrict__ offsets,
                   const int32_t* __restrict__ flat, const FwdItem* __restrict__ items,
                   const int32_t* __restrict__ n_items_ptr, float scale_log2, uint32_t tmem_cols, int kv_group,
                   __nv_bfloat16* __restrict__ part_o, float* __restrict__ part_lse) {
    using namespace sm100;
    constexpr int SL = D / 64;  // 64-wide slabs of the head dim
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* q_s = smem;                       // [SL][128][128B]
    uint8_t* k_s = q_s + kTcM * D * 2;         // [SL][BP][128B]
    uint8_t* v_s = k_s + BP * D * 2;           // [SL][BP][128B]
    uint8_t* p_s = v_s + BP * D * 2;           // [BP/64][128][128B]
    const int pslabs = (BP + 63) / 64;
    uint64_t* bars = reinterpret_cast<uint64_t*>(p_s + pslabs * kTcM * 128);
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(bars + 2);
    int32_t* qid_s = reinterpret_cast<int32_t*>(tmem_ptr + 4);

    const int tid = threadIdx.x, warp = tid >> 5;
    const int n_blocks = (int)((N + B - 1) / B);
    const int n_items = *n_items_ptr;
    const int per = (n_items + gridDim.x - 1) / gridDim.x;
    const int it0 = blockIdx.x * per;
    const int it1 = min(n_items, it0 + per);

    if (warp == 0) tmem_alloc(tmem_ptr, tmem_cols);
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_ptr;
    const uint32_t tmem_s = tmem;           // S: columns [0, BP)
    const uint32_t tmem_o = tmem + BP;      // O: columns [BP, BP + D)
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    const uint32_t idesc_s = idesc_bf16(kTcM, BP, false, false);
    const uint32_t idesc_o = idesc_bf16(kTcM, D, false, true);

    int cur_hj = -1;
    uint32_t phase = 0;
    for (int it = it0; it < it1; ++it) {
        const FwdItem item = items[it];
        const int64_t h = item.hj / n_blocks;
        const int j = item.hj % n_blocks;
        const int cnt = counts[item.hj];
        const int rows = min(kTcM, cnt - item.row0);
        const int64_t pbase = (int64_t)offsets[item.hj] + item.row0;
        const int64_t k0 = (int64_t)j * B;
        const int klen = (int)min64(B, N - k0);
        const __nv_bfloat16* Qh = Q + h * N * D;

        // ---- loads (all previous MMAs and TMEM reads finished: see the
        // barrier at the end of the previous iteration)
        const int q = (tid < rows) ? flat[h * N * width + pbase + tid] : -1;
        qid_s[tid] = q;
#pragma unroll
        for (int c = 0; c < D / 8; ++c) {
            const uint32_t dst = smem_u32(q_s) + sw128_off(tid, c * 8, kTcM);
            cp_async16(dst, Qh + (int64_t)max(q, 0) * D + c * 8, q >= 0);
        }
        if (item.hj != cur_hj) {
            cur_hj = item.hj;
            const __nv_bfloat16* Kh = K + ((h / kv_group) * N + k0) * D;   // GQA: K/V head of query head h
            const __nv_bfloat16* Vh = V + ((h / kv_group) * N + k0) * D;
            for (int e = tid; e < BP * (D / 8); e += 128) {
                const int r = e / (D / 8), c = e % (D / 8);
                const bool ok = r < klen;
                const uint32_t off = sw128_off(r, c * 8, BP);
                cp_async16(smem_u32(k_s) + off, Kh + (int64_t)(ok ? r : 0) * D + c * 8, ok);
                cp_async16(smem_u32(v_s) + off, Vh + (int64_t)(ok ? r : 0) * D + c * 8, ok);
            }
        }
        cp_async_commit();
        cp_async_wait<0>();
        fence_proxy_async_smem();
        __syncthreads();

        // ---- S = Q K^T
        if (tid == 0) {
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
                const int sl = kk >> 2, ke = (kk & 3) * 16;
                umma_bf16(tmem_s, desc_kmajor(smem_u32(q_s) + sl * kTcM * 128, ke),
                          desc_kmajor(smem_u32(k_s) + sl * BP * 128, ke), idesc_s, kk > 0);
            }
            umma_commit(&bars[0]);
        }
        mbar_wait(&bars[0], phase);
        tc_fence_after();

        // ---- softmax over the row (thread tid owns gathered row tid)
        const int64_t qq = q;
        float m = -INFINITY;
        for (int c0 = 0; c0 < BP; c0 += 32) {
            float sv[32];
            tmem_ld32(tmem_s + lane_off + c0, sv);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int col = c0 + i;
                const bool ok = col < klen && k0 + col <= qq;
                m = fmaxf(m, ok ? sv[i] * scale_log2 : -INFINITY);
            }
        }
        const float mref = (m == -INFINITY) ? 0.f : m;
        float l = 0.f;
        for (int c0 = 0; c0 < BP; c0 += 32) {
            float sv[32];
            tmem_ld32(tmem_s + lane_off + c0, sv);
            tmem_ld_wait();
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
                const int col = c0 + i;
                const float p0 = (col < klen && k0 + col <= qq) ? fast_exp2(sv[i] * scale_log2 - mref) : 0.f;
                const float p1 = (col + 1 < klen && k0 + col + 1 <= qq) ? fast_exp2(sv[i + 1] * scale_log2 - mref) : 0.f;
                l += p0 + p1;
                pk[i >> 1] = pack_bf16(p0, p1);
            }
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                const uint32_t off = sw128_off(tid, c0 + g * 8, kTcM);
                *reinterpret_cast<uint4*>(p_s + off) = make_uint4(pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
            }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncthreads();

        // ---- O = P V
        if (tid == 0) {
            tc_fence_after();
            for (int kk = 0; kk < BP / 16; ++kk) {
                const int sl = kk >> 2, ke = (kk & 3) * 16;
                umma_bf16(tmem_o, desc_kmajor(smem_u32(p_s) + sl * kTcM * 128, ke),
                          desc_mnmajor(smem_u32(v_s), kk * 16, BP * 128), idesc_o, kk > 0);
            }
            umma_commit(&bars[1]);
        }
        mbar_wait(&bars[1], phase);
        tc_fence_after();

        // ---- epilogue: normalised partial O (bf16) and its LSE. tcgen05.ld is
        // warp-collective: every lane loads, only rows of the tile store.
        {
            const float inv = 1.f / l;
            const bool live = tid < rows;
            __nv_bfloat16* po = part_o + (h * N * width + pbase + tid) * D;
#pragma unroll
            for (int c0 = 0; c0 < D; c0 += 32) {
                float ov[32];
                tmem_ld32(tmem_o + lane_off + c0, ov);
                tmem_ld_wait();
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(ov[2 * i] * inv, ov[2 * i + 1] * inv);
                if (live) {
#pragma unroll
                    for (int g = 0; g < 4; ++g)
                        *reinterpret_cast<uint4*>(po + c0 + g * 8) =
                            make_uint4(pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
                }
            }
            if (live) part_lse[h * N * width + pbase + tid] = (m + __log2f(l)) * kLn2;
        }
        tc_fence_before();
        __syncthreads();
        phase ^= 1;
    }
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, tmem_cols);
    }
}


// ---------------------------------------------------------------- warp-specialised tcgen05 path
// Persistent CTA, 6 warps, contiguous item range per CTA:
//   warp 0     producer: gathers the item's 128 query rows (cp.async,
//              completion tracked by mbarrier) and K_j / V_j when the block
//              changes; Q and K/V double buffered
//   warp 1     MMA issuer (one lane): S(i) = Q K^T into one of two TMEM S
//              buffers, O(i) = P(i) V into one of two TMEM O buffers, S(i+2)
//              issued right after O(i) so the tensor pipe always has work
//   warps 2-5  softmax + epilogue: row r = 32*(warp%4) + lane (TMEM lane
//              quadrant rule); softmax(i) from TMEM to bf16 P in smem, then
//              the epilogue of item i-1 (O from TMEM -> partial in HBM)
constexpr int kFwPr = 2;                    // producer (gather) warps
constexpr int kFwMma = kFwPr;               // MMA warp
constexpr int kWsThreads = 32 * (kFwPr + 1 + 4);

struct FwdWsBars {
    uint64_t q_full[2], q_empty[2], kv_full[2], kv_empty[2];
    uint64_t s_full[2], s_empty[2], p_full[2], p_empty[2], o_full[2], o_empty[2];
    uint32_t tmem;
};

template <int D>
__global__ void __launch_bounds__(kWsThreads, 1)
moba_fwd_ws_kernel(const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ K,
                   const __nv_bfloat16* __restrict__ V, int64_t N, int B, int BP, int width,
                   const int32_t* __restrict__ counts, const int32_t* __restrict__ offsets,
                   const int32_t* __restrict__ flat, const FwdItem* __restrict__ items,
                   const int32_t* __restrict__ n_items_ptr, float scale_log2, int q_stages,
                   __nv_bfloat16* __restrict__ part_o, float* __restrict__ part_lse) {
    using namespace sm100;
    constexpr uint32_t kTmemCols = 512;
    constexpr int kv_stages = 2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t q_bytes = kTcM * D * 2;
    const uint32_t kv_bytes = BP * D * 2;
    const uint32_t p_bytes = kTcM * 128 * ((BP + 63) / 64);
    uint8_t* q_s = smem;                                  // [q_stages][Q tile]
    uint8_t* kv_s = q_s + q_stages * q_bytes;             // [2][K tile | V tile]
    uint8_t* p_s = kv_s + kv_stages * 2 * kv_bytes;       // [2][P tile]
    FwdWsBars* bars = reinterpret_cast<FwdWsBars*>(p_s + 2 * p_bytes);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n_blocks = (int)((N + B - 1) / B);
    const int n_items = *n_items_ptr;
    const int per = (n_items + gridDim.x - 1) / gridDim.x;
    const int it0 = min(n_items, (int)blockIdx.x * per);
    const int it1 = min(n_items, it0 + per);
    const int n_local = it1 - it0;

    if (warp == kFwMma) tmem_alloc(&bars->tmem, kTmemCols);
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bars->q_full[s], 32 * kFwPr);
            mbar_init(&bars->q_empty[s], 1);
            mbar_init(&bars->kv_full[s], 32 * kFwPr);
            mbar_init(&bars->kv_empty[s], 1);
            mbar_init(&bars->s_full[s], 1);
            mbar_init(&bars->s_empty[s], 4);
            mbar_init(&bars->p_full[s], 4);
            mbar_init(&bars->p_empty[s], 1);
            mbar_init(&bars->o_full[s], 1);
            mbar_init(&bars->o_empty[s], 4);
        }
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem;

    if (n_local > 0) {
        if (warp < kFwPr) {
            // ------------------------------------------------ producers (coalesced gathers)
            int prev_hj = -1, kv_uses = -1;
            for (int li = 0; li < n_local; ++li) {
                const FwdItem item = items[it0 + li];
                const int64_t h = item.hj / n_blocks;
                const int j = item.hj % n_blocks;
                if (item.hj != prev_hj) {
                    prev_hj = item.hj;
                    ++kv_uses;
                    const int ks = kv_uses % kv_stages;
                    mbar_wait(&bars->kv_empty[ks], ((kv_uses / kv_stages) & 1) ^ 1);
                    const int64_t k0 = (int64_t)j * B;
                    const int klen = (int)min64(B, N - k0);
                    const __nv_bfloat16* Kh = K + (h * N + k0) * D;
                    const __nv_bfloat16* Vh = V + (h * N + k0) * D;
                    const uint32_t kb = smem_u32(kv_s + ks * 2 * kv_bytes);
                    for (int e = warp * 32 + lane; e < BP * (D / 8); e += 32 * kFwPr) {
                        const int r = e / (D / 8), c = e % (D / 8);
                        const bool ok = r < klen;
                        const uint32_t off = sw128_off(r, c * 8, BP);
                        cp_async16(kb + off, Kh + (int64_t)(ok ? r : 0) * D + c * 8, ok);
                        cp_async16(kb + kv_bytes + off, Vh + (int64_t)(ok ? r : 0) * D + c * 8, ok);
                    }
                    cpasync_arrive_noinc(&bars->kv_full[ks]);
                }
                const int qs = li % q_stages;
                mbar_wait(&bars->q_empty[qs], ((li / q_stages) & 1) ^ 1);
                const int rows = min(kTcM, counts[item.hj] - item.row0);
                const int32_t* fl = flat + h * N * width + offsets[item.hj] + item.row0;
                const __nv_bfloat16* Qh = Q + h * N * D;
                const uint32_t qb = smem_u32(q_s + qs * q_bytes);
                // 8 lanes per 128-B row segment: 4 rows per warp instruction
                const int sub = lane & 7, rsub = lane >> 3;
#pragma unroll
                for (int i = 0; i < kTcM / 4 / kFwPr; ++i) {
                    const int r = 4 * (warp + kFwPr * i) + rsub;
                    const int q = (r < rows) ? fl[r] : -1;
                    const __nv_bfloat16* src = Qh + (int64_t)max(q, 0) * D;
#pragma unroll
                    for (int c = sub; c < D / 8; c += 8) cp_async16(qb + sw128_off(r, c * 8, kTcM), src + c * 8, q >= 0);
                }
                cpasync_arrive_noinc(&bars->q_full[qs]);
            }
        } else if (warp == kFwMma) {
            // ------------------------------------------------ MMA issuer
            const uint32_t idesc_s = idesc_bf16(kTcM, BP, false, false);
            const uint32_t idesc_o = idesc_bf16(kTcM, D, false, true);
            int s_hj = -1, s_kv = -1;          // kv use counter as seen by the S stream
            int kv_of[2] = {0, 0};             // kv use index of the item in S buffer li&1
            auto issue_s = [&](int li) {
                const FwdItem item = items[it0 + li];
                if (item.hj != s_hj) {
                    s_hj = item.hj;
                    ++s_kv;
                    mbar_wait(&bars->kv_full[s_kv % kv_stages], (s_kv / kv_stages) & 1);
                }
                kv_of[li & 1] = s_kv;
                const int qs = li % q_stages;
                const int sb = li & 1;
                mbar_wait(&bars->q_full[qs], (li / q_stages) & 1);
                mbar_wait(&bars->s_empty[sb], ((li >> 1) & 1) ^ 1);
                tc_fence_after();
                fence_proxy_async_smem();
                if (lane == 0) {
                    const uint32_t qa = smem_u32(q_s + qs * q_bytes);
                    const uint32_t ka = smem_u32(kv_s + (s_kv % kv_stages) * 2 * kv_bytes);
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const int sl = kk >> 2, ke = (kk & 3) * 16;
                        umma_bf16(tmem + sb * BP, desc_kmajor(qa + sl * kTcM * 128, ke),
                                  desc_kmajor(ka + sl * BP * 128, ke), idesc_s, kk > 0);
                    }
                    umma_commit(&bars->s_full[sb]);
                    umma_commit(&bars->q_empty[qs]);
                }
                __syncwarp();
            };
            issue_s(0);
            if (n_local > 1) issue_s(1);
            for (int li = 0; li < n_local; ++li) {
                const int ps = li & 1;
                const int kvu = kv_of[ps];
                mbar_wait(&bars->p_full[ps], (li >> 1) & 1);
                mbar_wait(&bars->o_empty[ps], ((li >> 1) & 1) ^ 1);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t pa = smem_u32(p_s + ps * p_bytes);
                    const uint32_t va = smem_u32(kv_s + (kvu % kv_stages) * 2 * kv_bytes + kv_bytes);
                    for (int kk = 0; kk < BP / 16; ++kk) {
                        const int sl = kk >> 2, ke = (kk & 3) * 16;
                        umma_bf16(tmem + 2 * BP + ps * D, desc_kmajor(pa + sl * kTcM * 128, ke),
                                  desc_mnmajor(va, kk * 16, BP * 128), idesc_o, kk > 0);
                    }
                    umma_commit(&bars->o_full[ps]);
                    umma_commit(&bars->p_empty[ps]);
                    const bool last_use = (li + 1 == n_local) || items[it0 + li + 1].hj != items[it0 + li].hj;
                    if (last_use) umma_commit(&bars->kv_empty[kvu % kv_stages]);
                }
                __syncwarp();
                if (li + 2 < n_local) issue_s(li + 2);
            }
        } else {
            // ------------------------------------------------ softmax + epilogue
            const int row = 32 * (warp & 3) + lane;
            const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
            float l_prev = 1.f, m_prev = 0.f;
            int64_t p_prev = 0;
            bool live_prev = false;
            for (int li = 0; li <= n_local; ++li) {
                float l_cur = 1.f, m_cur = 0.f;
                int64_t p_cur = 0;
                bool live_cur = false;
                if (li < n_local) {
                    const FwdItem item = items[it0 + li];
                    const int64_t h = item.hj / n_blocks;
                    const int j = item.hj % n_blocks;
                    const int rows = min(kTcM, counts[item.hj] - item.row0);
                    const int64_t pb = (int64_t)offsets[item.hj] + item.row0;
                    live_cur = row < rows;
                    const int64_t q = live_cur ? flat[h * N * width + pb + row] : -1;
                    const int64_t k0 = (int64_t)j * B;
                    const int klen = (int)min64(B, N - k0);
                    // visible keys of this row: col < lim
                    const int lim = (int)min64(klen, q - k0 + 1);
                    p_cur = h * N * width + pb + row;
                    const int sb = li & 1;
                    mbar_wait(&bars->s_full[sb], (li >> 1) & 1);
                    tc_fence_after();
                    float sv[4][32];
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (c * 32 < BP) tmem_ld32(tmem + sb * BP + lane_off + c * 32, sv[c]);
                    tmem_ld_wait();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&bars->s_empty[sb]);
                    float m = -INFINITY;
#pragma unroll
                    for (int c = 0; c < 4; ++c)
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            const bool ok = c * 32 + i < lim;
                            sv[c][i] = ok ? sv[c][i] * scale_log2 : -INFINITY;
                            m = fmaxf(m, sv[c][i]);
                        }
                    const float mref = (m == -INFINITY) ? 0.f : m;
                    float l = 0.f;
                    mbar_wait(&bars->p_empty[sb], ((li >> 1) & 1) ^ 1);
                    const uint32_t pt = smem_u32(p_s) + sb * p_bytes;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        if (c * 32 < BP) {
                            uint32_t pk[16];
#pragma unroll
                            for (int i = 0; i < 32; i += 2) {
                                const float p0 = fast_exp2(sv[c][i] - mref);
                                const float p1 = fast_exp2(sv[c][i + 1] - mref);
                                l += p0 + p1;
                                pk[i >> 1] = pack_bf16(p0, p1);
                            }
#pragma unroll
                            for (int g = 0; g < 4; ++g)
                                sts128(pt + sw128_off(row, c * 32 + g * 8, kTcM),
                                       make_uint4(pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]));
                        }
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&bars->p_full[sb]);
                    l_cur = l;
                    m_cur = m;
                }
                if (li >= 1) {
                    // epilogue of item li-1
                    const int ob = (li - 1) & 1;
                    mbar_wait(&bars->o_full[ob], ((li - 1) >> 1) & 1);
                    tc_fence_after();
                    const float inv = 1.f / l_prev;
                    __nv_bfloat16* po = part_o + p_prev * D;
#pragma unroll
                    for (int c0 = 0; c0 < D; c0 += 32) {
                        float ov[32];
                        tmem_ld32(tmem + 2 * BP + ob * D + lane_off + c0, ov);
                        tmem_ld_wait();
                        if (live_prev) {
                            uint32_t pk[16];
#pragma unroll
                            for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(ov[2 * i] * inv, ov[2 * i + 1] * inv);
#pragma unroll
                            for (int g = 0; g < 4; ++g)
                                *reinterpret_cast<uint4*>(po + c0 + g * 8) =
                                    make_uint4(pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&bars->o_empty[ob]);
                    if (live_prev) part_lse[p_prev] = (m_prev + __log2f(l_prev)) * kLn2;
                }
                l_prev = l_cur;
                m_prev = m_cur;
                p_prev = p_cur;
                live_prev = live_cur;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kFwMma) {
        tc_fence_after();
        tmem_dealloc(tmem, kTmemCols);
    }
}

// ---------------------------------------------------------------- combine
#ifndef MOBA_COMBINE_QW
#define MOBA_COMBINE_QW 1   // one query per warp: fewer registers, more warps in flight (64K combine 0.78 -> 0.62 ms vs 2)
#endif
// One warp per query: merge its <= width partials (lse-weighted,
// SoftmaxState.finalize over the query's blocks, src/attention.py:70-74).
// A partial row (D bf16) is read by L = D/8 lanes with 16-B loads, so one
// warp instruction fetches 32/L partial rows; all rounds are issued before
// any is consumed. The lane groups are then reduced with shuffles and the
// first L lanes write the row (coalesced).
template <int D, int WMAX, int slabs>
__global__ void __launch_bounds__(256)
moba_combine_kernel(const __nv_bfloat16* __restrict__ part_o, const float* __restrict__ part_lse,
                    const int32_t* __restrict__ row_pos, int64_t N, int width, int64_t total_rows,
                    __nv_bfloat16* __restrict__ O, float* __restrict__ LSE) {
    // a query's partials: (slot, slab) pairs, virtual slot v = slot * slabs + slab
    // at partial position row_pos[slot] * slabs + slab (slabs = 1 unless the
    // key blocks are longer than 128)
    const int vwidth = width * slabs;
    constexpr int L = D / 8;               // lanes per partial row
    constexpr int G = 32 / L;              // partial rows per warp instruction
    constexpr int R = (WMAX + G - 1) / G;  // load rounds per query
    constexpr int QW = MOBA_COMBINE_QW;    // queries per warp, loads of all in flight together
    const int64_t row0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * QW;
    const int lane = threadIdx.x & 31;
    if (row0 >= total_rows) return;
    const int grp = lane / L, sub = lane % L;
    int32_t p[QW];
#pragma unroll
    for (int t = 0; t < QW; ++t)
    {
        const int32_t q = (lane < vwidth && row0 + t < total_rows) ? __ldg(row_pos + (row0 + t) * width + lane / slabs) : -1;
        p[t] = q >= 0 ? q * slabs + lane % slabs : -1;
    }
    float ls[QW];
    uint4 raw[QW][R];
    int32_t pr[QW][R];
#pragma unroll
    for (int t = 0; t < QW; ++t) {
        const int64_t h = (row0 + t) / N;
        ls[t] = (p[t] >= 0) ? __ldg(part_lse + h * N * vwidth + p[t]) : -INFINITY;
        const uint4* base = reinterpret_cast<const uint4*>(part_o + h * N * vwidth * D) + sub;
        const int32_t p0 = max(__shfl_sync(0xffffffffu, p[t], 0), 0);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            pr[t][r] = __shfl_sync(0xffffffffu, p[t], (r * G + grp) & 31);
            if (r * G + grp >= vwidth) pr[t][r] = -1;
            raw[t][r] = __ldg(base + (int64_t)(pr[t][r] >= 0 ? pr[t][r] : p0) * L);
        }
    }
#pragma unroll
    for (int t = 0; t < QW; ++t) {
        const int64_t row = row0 + t;
        const float m = warp_max(ls[t]);
        const float w = (p[t] >= 0) ? __expf(ls[t] - m) : 0.f;
        const float wsum = warp_sum(w);
        float acc[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = 0.f;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            float wt = __shfl_sync(0xffffffffu, w, (r * G + grp) & 31);
            if (pr[t][r] < 0) wt = 0.f;
            const uint32_t u[4] = {raw[t][r].x, raw[t][r].y, raw[t][r].z, raw[t][r].w};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float2 f = unpack_bf16(u[c]);
                acc[2 * c] = fmaf(wt, f.x, acc[2 * c]);
                acc[2 * c + 1] = fmaf(wt, f.y, acc[2 * c + 1]);
            }
        }
#pragma unroll
        for (int o = L; o < 32; o <<= 1)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
        if (row < total_rows) {
            const float inv = 1.f / wsum;
            if (grp == 0) {
                uint4 outv = make_uint4(pack_bf16(acc[0] * inv, acc[1] * inv), pack_bf16(acc[2] * inv, acc[3] * inv),
                                        pack_bf16(acc[4] * inv, acc[5] * inv), pack_bf16(acc[6] * inv, acc[7] * inv));
                *(reinterpret_cast<uint4*>(O + row * D) + sub) = outv;
            }
            if (lane == 0) LSE[row] = m + __logf(wsum);
        }
    }
}

template <int D>
static void launch_combine(const void* part_o, const float* part_lse, const int32_t* row_pos, int64_t N, int width,
                           int64_t rows, void* out, float* lse, cudaStream_t s, int slabs = 1) {
    const unsigned grid = (unsigned)ceil_div(rows, 8 * MOBA_COMBINE_QW);
    auto po = (const __nv_bfloat16*)part_o;
    auto o = (__nv_bfloat16*)out;
#define MOBA_COMBINE(W, S) moba_combine_kernel<D, W, S><<<grid, 256, 0, s>>>(po, part_lse, row_pos, N, width, rows, o, lse)
#define MOBA_COMBINE_W(S)                                \
    do {                                                 \
        const int vw = width * (S);                      \
        if (vw <= 4) MOBA_COMBINE(4, S);                 \
        else if (vw <= 8) MOBA_COMBINE(8, S);            \
        else if (vw <= 12) MOBA_COMBINE(12, S);          \
        else if (vw <= 16) MOBA_COMBINE(16, S);          \
        else if (vw <= 24) MOBA_COMBINE(24, S);          \
        else MOBA_COMBINE(32, S);                        \
    } while (0)
    if (slabs == 1) MOBA_COMBINE_W(1);
    else if (slabs == 2) MOBA_COMBINE_W(2);
    else if (slabs == 3) MOBA_COMBINE_W(3);
    else MOBA_COMBINE_W(4);
#undef MOBA_COMBINE_W
#undef MOBA_COMBINE
}

// ---------------------------------------------------------------- work items
// One thread per (head, block): exclusive scan of tile counts in a single
// CTA, then each (head, block) writes its items.
__global__ void __launch_bounds__(1024)
fwd_items_scan_kernel(const int32_t* __restrict__ counts, int64_t total, int bm, int mult,
                      int32_t* __restrict__ item_off, int32_t* __restrict__ n_items) {
    __shared__ int32_t warp_tot[32];
    __shared__ int32_t carry;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t b0 = 0; b0 < total; b0 += 1024) {
        int64_t b = b0 + threadIdx.x;
        int32_t v = (b < total) ? (counts[b] + bm - 1) / bm * mult : 0;
        int32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_tot[wid] = x;
        __syncthreads();
        if (wid == 0) {
            int32_t t = warp_tot[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int32_t y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += y;
            }
            warp_tot[lane] = t;
        }
        __syncthreads();
        if (b < total) item_off[b] = carry + (wid ? warp_tot[wid - 1] : 0) + x - v;
        __syncthreads();
        if (threadIdx.x == 0) carry += warp_tot[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) *n_items = carry;
}

__global__ void fwd_items_fill_kernel(const int32_t* __restrict__ counts, const int32_t* __restrict__ item_off,
                                      int64_t total, int bm, FwdItem* __restrict__ items) {
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= total) return;
    int nt = (counts[b] + bm - 1) / bm;
    int32_t o = item_off[b];
    for (int t = 0; t < nt; ++t) items[o + t] = FwdItem{(int32_t)b, t * bm};
}

// workspace layout (all head-local regions back to back):
//   part_o   bf16 [bh, N*width, D]
//   part_lse f32  [bh, N*width]
//   item_off i32  [bh*n]
//   n_items  i32
//   items    FwdItem [bh*(ceil(N*width/BM) + n)]
size_t fwd_ts_item_bytes();

struct FwdWs {
    size_t part_o, part_lse, item_off, n_items, items, total;
};

// key-block slabs of the ping-pong forward: blocks longer than 128 keys are
// processed as ceil(B / 128) slabs, each with its own partial
static int fwd_slabs(int B) { return (int)ceil_div(B, 128); }

static FwdWs fwd_ws_layout(int64_t bh, int64_t N, int D, int B, int width) {
    FwdWs w;
    int64_t n = ceil_div(N, B);
    int64_t E = N * width * fwd_slabs(B);
    size_t off = 0;
    w.part_o = off;
    off = align_up(off + (size_t)bh * E * D * 2, 256);
    w.part_lse = off;
    off = align_up(off + (size_t)bh * E * 4, 256);
    w.item_off = off;
    off = align_up(off + (size_t)bh * n * 4, 256);
    w.n_items = off;
    off = align_up(off + 4, 256);
    w.items = off;
    off = align_up(off + (size_t)bh * (ceil_div(E, kFwdBM) + n * fwd_slabs(B)) *
                             std::max(sizeof(FwdItem), fwd_ts_item_bytes()), 256);
    w.total = off;
    return w;
}

template <int D>
int launch_fwd_ts(const void* q, const void* k, const void* v, int64_t bh, int kv_group, int64_t N, int B, int width,
                  const int32_t* flat, const void* items, const int32_t* item_lo, const int32_t* item_hi,
                  float scale_log2, void* part_o, float* part_lse, cudaStream_t s);
void fwd_ts_fill_items(const int32_t* counts, const int32_t* offsets, const int32_t* item_off, int64_t total,
                       int slabs, void* items, cudaStream_t s);
size_t fwd_ts_item_bytes();

template <int D>
static int launch_fwd(const void* q, const void* k, const void* v, int64_t bh, int kv_group, int64_t N, int B,
                      int width, const int32_t* counts, const int32_t* offsets, const int32_t* flat,
                      const int32_t* row_pos, float scale, void* out, float* lse, uint8_t* ws, const FwdWs& L,
                      cudaStream_t s) {
    const int64_t n = ceil_div(N, B);
    const int64_t total = bh * n;
    int32_t* item_off = (int32_t*)(ws + L.item_off);
    int32_t* n_items = (int32_t*)(ws + L.n_items);
    FwdItem* items = (FwdItem*)(ws + L.items);
    const char* impl = std::getenv("MOBA_FWD_IMPL");
    const bool use_mma = impl != nullptr && impl[0] == 'm';
    const int S = fwd_slabs(B);
    const bool use_ts = (impl == nullptr || impl[0] == 't') && width * S <= 32;
    // GQA (kv_group > 1) is wired into the default kernels (ping-pong ts for
    // B <= 128, simple tcgen05 above); the legacy variants are MHA only
    if (kv_group > 1 && (use_mma || (!use_ts && ceil_div(B, 16) * 16 <= 128))) return MOBA_ERR_UNSUPPORTED;
    const int bm = use_mma ? kFwdBM : kTcM;
    fwd_items_scan_kernel<<<1, 1024, 0, s>>>(counts, total, bm, use_ts ? S : 1, item_off, n_items);
    if (!use_ts) fwd_items_fill_kernel<<<(unsigned)ceil_div(total, 256), 256, 0, s>>>(counts, item_off, total, bm, items);
    int st = check_launch("fwd_items", use_ts ? 1 : 2);
    if (st) return st;
    const int64_t max_items = bh * (ceil_div(N * width, bm) + n);
    if (use_ts) {
        // heads in chunks whose partials (<= 48 MB) stay in L2 until the
        // chunk's combine reads them back
        fwd_ts_fill_items(counts, offsets, item_off, total, S, items, s);
        st = check_launch("fwd_ts_items_kernel");
        if (st) return st;
        const int64_t per_head = N * width * (int64_t)S * D * 2;
        // (measured: smaller fwd launches cost more in pipeline ramp-up than the
        // combine saves, so by default all heads form one chunk)
        const char* chunk_env = std::getenv("MOBA_FWD_CHUNK_MB");
        const int64_t chunk_mb = chunk_env ? std::atoll(chunk_env) : 0;
        const int64_t hc = chunk_mb > 0 ? std::max<int64_t>(1, (chunk_mb << 20) / per_head) : bh;
        for (int64_t h0 = 0; h0 < bh; h0 += hc) {
            const int64_t h1 = std::min(bh, h0 + hc);
            const int32_t* lo = item_off + h0 * n;
            const int32_t* hi = h1 < bh ? item_off + h1 * n : n_items;
            st = launch_fwd_ts<D>(q, k, v, bh, kv_group, N, B, width, flat, items, lo, hi, scale * kLog2e, ws + L.part_o,
                                  (float*)(ws + L.part_lse), s);
            if (st) return st;
            StageTimer tm(T_COMBINE, s);
            launch_combine<D>(ws + L.part_o + h0 * N * width * S * D * 2,
                              (const float*)(ws + L.part_lse) + h0 * N * width * S, row_pos + h0 * N * width, N, width,
                              (h1 - h0) * N, (uint8_t*)out + h0 * N * D * 2, lse + h0 * N, s, S);
            st = check_launch("moba_combine_kernel");
            if (st) return st;
        }
        return MOBA_OK;
    } else if (use_mma) {
        const int BP = (int)ceil_div(B, 64) * 64;
        const size_t smem = (size_t)(kFwdBM + 2 * BP) * D * 2 + kFwdBM * 4;
        auto kern = moba_fwd_mma_kernel<D>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kFwdThreads, smem);
        if (occ < 1) return MOBA_ERR_UNSUPPORTED;
        const int grid = (int)std::min<int64_t>(max_items, (int64_t)kNumSMs * occ);
        StageTimer tm(T_FWD, s);
        kern<<<grid, kFwdThreads, smem, s>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
                                             (const __nv_bfloat16*)v, N, B, BP, width, counts, offsets, flat, items,
                                             n_items, scale * kLog2e, (__nv_bfloat16*)(ws + L.part_o),
                                             (float*)(ws + L.part_lse));
    } else if (ceil_div(B, 16) * 16 <= 128 && !(impl != nullptr && impl[0] == 's')) {
        const int BP = (int)ceil_div(B, 16) * 16;
        const size_t q_bytes = (size_t)kTcM * D * 2, kv_bytes = (size_t)BP * D * 2;
        const size_t p_bytes = (size_t)kTcM * 128 * ((BP + 63) / 64);
        int q_stages = 2;
        size_t smem = 1024 + q_stages * q_bytes + 2 * 2 * kv_bytes + 2 * p_bytes + sizeof(FwdWsBars);
        if (smem > 232448) {
            q_stages = 1;
            smem = 1024 + q_bytes + 2 * 2 * kv_bytes + 2 * p_bytes + sizeof(FwdWsBars);
        }
        if (smem > 232448) return MOBA_ERR_UNSUPPORTED;
        auto kern = moba_fwd_ws_kernel<D>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int grid = (int)std::min<int64_t>(max_items, (int64_t)kNumSMs);
        StageTimer tm(T_FWD, s);
        kern<<<grid, kWsThreads, smem, s>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
                                            (const __nv_bfloat16*)v, N, B, BP, width, counts, offsets, flat, items,
                                            n_items, scale * kLog2e, q_stages, (__nv_bfloat16*)(ws + L.part_o),
                                            (float*)(ws + L.part_lse));
    } else {
        const int BP = (int)ceil_div(B, 16) * 16;
        const int pslabs = (BP + 63) / 64;
        const size_t smem = 1024 + (size_t)kTcM * D * 2 + 2 * (size_t)BP * D * 2 + (size_t)pslabs * kTcM * 128 +
                            64 + kTcM * 4;
        uint32_t cols = 32;
        while (cols < (uint32_t)(BP + D)) cols <<= 1;
        if (cols > 512 || smem > 232448) return MOBA_ERR_UNSUPPORTED;
        auto kern = moba_fwd_tc_kernel<D>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, smem);
        occ = std::min<int>(occ, (int)(512 / cols));
        if (occ < 1) return MOBA_ERR_UNSUPPORTED;
        const int grid = (int)std::min<int64_t>(max_items, (int64_t)kNumSMs * occ);
        StageTimer tm(T_FWD, s);
        kern<<<grid, 128, smem, s>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k, (const __nv_bfloat16*)v, N, B,
                                     BP, width, counts, offsets, flat, items, n_items, scale * kLog2e, cols, kv_group,
                                     (__nv_bfloat16*)(ws + L.part_o), (float*)(ws + L.part_lse));
    }
    st = check_launch("moba_fwd_kernel");
    if (st) return st;
    StageTimer tm(T_COMBINE, s);
    const int64_t rows = bh * N;
    launch_combine<D>(ws + L.part_o, (const float*)(ws + L.part_lse), row_pos, N, width, rows, out, lse, s);
    return check_launch("moba_combine_kernel");
}

}  // namespace moba

using namespace moba;

extern "C" size_t moba_fwd_workspace_size(int64_t bh, int64_t n_tokens, int head_dim, int block_size, int width) {
    if (bh < 1 || n_tokens < 1 || block_size < 1 || width < 1) return 0;
    return fwd_ws_layout(bh, n_tokens, head_dim, block_size, width).total;
}

extern "C" int moba_fwd_gqa(const void* q, const void* k, const void* v, int64_t bh, int kv_group, int64_t n_tokens,
                            int head_dim, int block_size, int width, const int32_t* counts, const int32_t* offsets,
                            const int32_t* flat, const int32_t* row_pos, float softmax_scale, void* out, float* lse,
                            void* workspace, size_t workspace_bytes, void* stream) {
    if (bh < 1 || n_tokens < 1 || block_size < 1 || width < 1) return MOBA_ERR_SHAPE;
    if (kv_group < 1 || bh % kv_group != 0) return MOBA_ERR_SHAPE;
    if (width > 32 || block_size > 512) return MOBA_ERR_UNSUPPORTED;
    if (n_tokens * width >= (1ll << 31)) return MOBA_ERR_UNSUPPORTED;
    FwdWs L = fwd_ws_layout(bh, n_tokens, head_dim, block_size, width);
    if (workspace_bytes < L.total) return MOBA_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t* ws = (uint8_t*)workspace;
    if (head_dim == 64)
        return launch_fwd<64>(q, k, v, bh, kv_group, n_tokens, block_size, width, counts, offsets, flat, row_pos,
                              softmax_scale, out, lse, ws, L, s);
    if (head_dim == 128)
        return launch_fwd<128>(q, k, v, bh, kv_group, n_tokens, block_size, width, counts, offsets, flat, row_pos,
                               softmax_scale, out, lse, ws, L, s);
    return MOBA_ERR_UNSUPPORTED;
}

extern "C" int moba_fwd(const void* q, const void* k, const void* v, int64_t bh, int64_t n_tokens, int head_dim,
                        int block_size, int width, const int32_t* counts, const int32_t* offsets,
                        const int32_t* flat, const int32_t* row_pos, float softmax_scale, void* out, float* lse,
                        void* workspace, size_t workspace_bytes, void* stream) {
    return moba_fwd_gqa(q, k, v, bh, 1, n_tokens, head_dim, block_size, width, counts, offsets, flat, row_pos,
                        softmax_scale, out, lse, workspace, workspace_bytes, stream);
}
