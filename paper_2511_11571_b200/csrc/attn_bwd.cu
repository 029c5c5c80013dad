// Backward: key-block-major recomputation (moba_backward,
// src/attention.py:239-302; paper Alg. 5).
//
//   bwd_preprocess : D = rowsum(dO * O) (src/attention.py:266), zero dQ_acc
//   bwd main       : one CTA per (head, key block, <=128-key slab). K_j/V_j
//                    stay in shared memory; the CTA walks the block's varlen
//                    slice in 64-query tiles, gathers Q/dO/L/D, recomputes
//                    S and P = exp(S - L) (src/attention.py:229), and
//                    accumulates dV_j += P^T dO, dK_j += dS^T Q in registers
//                    (src/attention.py:230-233); dQ += dS K_j goes to an
//                    fp32 accumulator with vector reductions
//                    (src/attention.py:234).
//   bwd_finalize   : dQ = dQ_acc * scale -> bf16 (src/attention.py:299)
//
// This is the legacy-MMA (mma.sync m16n8k16) path.
#include "common.cuh"

namespace moba {

constexpr int kBwdBM = 64;  // gathered queries per tile
constexpr float kLog2eB = 1.4426950408889634f;

template <int D, int KT>
__global__ void __launch_bounds__(KT * 2)
moba_bwd_mma_kernel(const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ K,
                    const __nv_bfloat16* __restrict__ V, const __nv_bfloat16* __restrict__ dO,
                    const float* __restrict__ lse, const float* __restrict__ Dd, int64_t N, int B, int width,
                    const int32_t* __restrict__ counts, const int32_t* __restrict__ offsets,
                    const int32_t* __restrict__ flat, float scale, float* __restrict__ dq_acc,
                    float* __restrict__ dq_part, int64_t part_stride,
                    __nv_bfloat16* __restrict__ dK, __nv_bfloat16* __restrict__ dV) {
    constexpr int RB = D * 2;
    constexpr int CH = D / 8;
    constexpr int NW = KT / 16;          // warps: 16 keys each
    constexpr int NT = NW * 32;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* k_s = smem;
    uint8_t* v_s = k_s + KT * RB;
    uint8_t* q_s = v_s + KT * RB;
    uint8_t* do_s = q_s + kBwdBM * RB;
    uint8_t* ds_s = do_s + kBwdBM * RB;  // [KT keys][64 queries] bf16, 128 B rows
    float* l_s = reinterpret_cast<float*>(ds_s + KT * 128);
    float* d_s = l_s + kBwdBM;
    int32_t* qid_s = reinterpret_cast<int32_t*>(d_s + kBwdBM);

    const int n_blocks = (int)((N + B - 1) / B);
    const int slabs = (B + KT - 1) / KT;
    const int j = blockIdx.x / slabs;
    const int slab = blockIdx.x % slabs;
    const int64_t h = blockIdx.y;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, t4 = lane & 3;

    const int64_t kb0 = (int64_t)j * B + slab * KT;           // first key of the slab
    const int klen = (int)max64(0, min64(min64((int64_t)KT, (int64_t)B - slab * KT), N - kb0));
    const int hj = (int)(h * n_blocks + j);
    const int cnt = counts[hj];
    const int32_t* fl = flat + h * N * width + offsets[hj];
    const __nv_bfloat16* Qh = Q + h * N * D;
    const __nv_bfloat16* dOh = dO + h * N * D;

    for (int e = tid; e < KT * CH; e += NT) {
        int r = e / CH, c = e % CH;
        bool ok = r < klen;
        int64_t src = (h * N + kb0 + (ok ? r : 0)) * D + c * 8;
        cp_async16(smem_u32(k_s + swz<RB>(r, c)), K + src, ok);
        cp_async16(smem_u32(v_s + swz<RB>(r, c)), V + src, ok);
    }
    cp_async_commit();

    const int m0 = warp * 16;  // this warp's keys within the slab
    float dk[D / 8][4], dv[D / 8][4];
#pragma unroll
    for (int nt = 0; nt < D / 8; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) dk[nt][e] = dv[nt][e] = 0.f;

    const float sl2 = scale * kLog2eB;
    for (int r0 = 0; r0 < cnt; r0 += kBwdBM) {
        const int rows = min(kBwdBM, cnt - r0);
        __syncthreads();  // previous tile fully consumed
        if (tid < kBwdBM) {
            int qi = (tid < rows) ? fl[r0 + tid] : -1;
            qid_s[tid] = qi;
            l_s[tid] = (qi >= 0) ? lse[h * N + qi] * kLog2eB : 0.f;
            d_s[tid] = (qi >= 0) ? Dd[h * N + qi] : 0.f;
        }
        __syncthreads();
        for (int e = tid; e < kBwdBM * CH; e += NT) {
            int r = e / CH, c = e % CH;
            int qi = qid_s[r];
            int64_t src = (int64_t)max(qi, 0) * D + c * 8;
            cp_async16(smem_u32(q_s + swz<RB>(r, c)), Qh + src, qi >= 0);
            cp_async16(smem_u32(do_s + swz<RB>(r, c)), dOh + src, qi >= 0);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();

        // ---- S^T = K_w Q^T  (16 keys x 64 queries) and dP^T = V_w dO^T
        float s[8][4], dp[8][4];
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) s[nt][e] = dp[nt][e] = 0.f;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
            uint32_t ka[4], va[4];
            {
                int r = m0 + (lane & 7) + ((lane >> 3) & 1) * 8;
                int c = kk * 2 + (lane >> 4);
                ldmatrix_x4(smem_u32(k_s + swz<RB>(r, c)), ka[0], ka[1], ka[2], ka[3]);
                ldmatrix_x4(smem_u32(v_s + swz<RB>(r, c)), va[0], va[1], va[2], va[3]);
            }
#pragma unroll
            for (int np = 0; np < 4; ++np) {
                int r = np * 16 + (lane & 7) + (lane >> 4) * 8;
                int c = kk * 2 + ((lane >> 3) & 1);
                uint32_t b0, b1, b2, b3;
                ldmatrix_x4(smem_u32(q_s + swz<RB>(r, c)), b0, b1, b2, b3);
                mma_bf16_16816(s[2 * np], ka, b0, b1);
                mma_bf16_16816(s[2 * np + 1], ka, b2, b3);
                ldmatrix_x4(smem_u32(do_s + swz<RB>(r, c)), b0, b1, b2, b3);
                mma_bf16_16816(dp[2 * np], va, b0, b1);
                mma_bf16_16816(dp[2 * np + 1], va, b2, b3);
            }
        }
        // ---- P^T, dS^T (element: key row m0+g(+8), query col nt*8+2t4(+1))
        const int key_lo = m0 + g, key_hi = m0 + g + 8;
        uint32_t pa[4][4], dsa[4][4];
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
            float pv[4], dsv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                int qc = nt * 8 + 2 * t4 + (e & 1);
                int key = (e < 2) ? key_lo : key_hi;
                int qi = qid_s[qc];
                bool ok = qi >= 0 && key < klen && (kb0 + key) <= (int64_t)qi;
                float p = ok ? fast_exp2(s[nt][e] * sl2 - l_s[qc]) : 0.f;
                pv[e] = p;
                dsv[e] = p * (dp[nt][e] - d_s[qc]);
            }
            pa[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16(pv[0], pv[1]);
            pa[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16(pv[2], pv[3]);
            dsa[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16(dsv[0], dsv[1]);
            dsa[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16(dsv[2], dsv[3]);
            // dS^T to smem for the dQ product: row = key, col = query
            *reinterpret_cast<uint32_t*>(ds_s + swz<128>(key_lo, nt) + 4 * t4) = dsa[nt >> 1][(nt & 1) * 2 + 0];
            *reinterpret_cast<uint32_t*>(ds_s + swz<128>(key_hi, nt) + 4 * t4) = dsa[nt >> 1][(nt & 1) * 2 + 1];
        }
        // ---- dV += P^T dO ; dK += dS^T Q   (k = query)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
            for (int np = 0; np < D / 16; ++np) {
                int r = ks * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
                int c = np * 2 + (lane >> 4);
                uint32_t b0, b1, b2, b3;
                ldmatrix_x4_trans(smem_u32(do_s + swz<RB>(r, c)), b0, b1, b2, b3);
                mma_bf16_16816(dv[2 * np], pa[ks], b0, b1);
                mma_bf16_16816(dv[2 * np + 1], pa[ks], b2, b3);
                ldmatrix_x4_trans(smem_u32(q_s + swz<RB>(r, c)), b0, b1, b2, b3);
                mma_bf16_16816(dk[2 * np], dsa[ks], b0, b1);
                mma_bf16_16816(dk[2 * np + 1], dsa[ks], b2, b3);
            }
        }
        __syncthreads();  // ds_s complete
        // ---- dQ (64 q x D) += dS (64 q x KT keys) K_slab (KT x D)
        {
            constexpr int QW = 4;                    // 16-query row groups
            constexpr int DSPLIT = NW / QW;          // d splits across warps
            constexpr int DW = D / DSPLIT;           // d columns per warp
            const int qr = (warp % QW) * 16;
            const int dc0 = (warp / QW) * DW;
            float acc[DW / 8][4];
#pragma unroll
            for (int nt = 0; nt < DW / 8; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
#pragma unroll
            for (int kk = 0; kk < KT / 16; ++kk) {
                uint32_t a[4];
                {
                    int key = kk * 16 + (lane & 7) + (lane >> 4) * 8;
                    int qc = (qr >> 3) + ((lane >> 3) & 1);
                    ldmatrix_x4_trans(smem_u32(ds_s + swz<128>(key, qc)), a[0], a[1], a[2], a[3]);
                }
#pragma unroll
                for (int np = 0; np < DW / 16; ++np) {
                    int key = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
                    int c = (dc0 >> 3) + np * 2 + (lane >> 4);
                    uint32_t b0, b1, b2, b3;
                    ldmatrix_x4_trans(smem_u32(k_s + swz<RB>(key, c)), b0, b1, b2, b3);
                    mma_bf16_16816(acc[2 * np], a, b0, b1);
                    mma_bf16_16816(acc[2 * np + 1], a, b2, b3);
                }
            }
            const int q_lo = qid_s[qr + g], q_hi = qid_s[qr + g + 8];
            if (dq_part != nullptr) {
                // deterministic schedule: one partial per (query, block,
                // slab) at its flat position, summed in slot order later
                float* dst = dq_part + slab * part_stride +
                             (h * N * width + offsets[hj] + r0 + qr) * (int64_t)D;
#pragma unroll
                for (int nt = 0; nt < DW / 8; ++nt) {
                    int col = dc0 + nt * 8 + 2 * t4;
                    if (q_lo >= 0)
                        *reinterpret_cast<float2*>(dst + (int64_t)g * D + col) = make_float2(acc[nt][0], acc[nt][1]);
                    if (q_hi >= 0)
                        *reinterpret_cast<float2*>(dst + (int64_t)(g + 8) * D + col) =
                            make_float2(acc[nt][2], acc[nt][3]);
                }
            } else {
#pragma unroll
                for (int nt = 0; nt < DW / 8; ++nt) {
                    int col = dc0 + nt * 8 + 2 * t4;
                    if (q_lo >= 0) red_add_f32x2(dq_acc + (h * N + q_lo) * D + col, acc[nt][0], acc[nt][1]);
                    if (q_hi >= 0) red_add_f32x2(dq_acc + (h * N + q_hi) * D + col, acc[nt][2], acc[nt][3]);
                }
            }
        }
    }
    cp_async_wait<0>();  // (no-op when the slice was non-empty)
    // ---- write dK_j = scale * dK, dV_j
    const int key_lo = m0 + g, key_hi = m0 + g + 8;
#pragma unroll
    for (int nt = 0; nt < D / 8; ++nt) {
        int col = nt * 8 + 2 * t4;
        if (key_lo < klen) {
            int64_t o = (h * N + kb0 + key_lo) * D + col;
            *reinterpret_cast<uint32_t*>(dK + o) = pack_bf16(dk[nt][0] * scale, dk[nt][1] * scale);
            *reinterpret_cast<uint32_t*>(dV + o) = pack_bf16(dv[nt][0], dv[nt][1]);
        }
        if (key_hi < klen) {
            int64_t o = (h * N + kb0 + key_hi) * D + col;
            *reinterpret_cast<uint32_t*>(dK + o) = pack_bf16(dk[nt][2] * scale, dk[nt][3] * scale);
            *reinterpret_cast<uint32_t*>(dV + o) = pack_bf16(dv[nt][2], dv[nt][3]);
        }
    }
}

// D = rowsum(dO * O) and dq_acc = 0; one warp per row.
template <int D>
__global__ void bwd_preprocess_kernel(const __nv_bfloat16* __restrict__ O, const __nv_bfloat16* __restrict__ dO,
                                      int64_t rows, float* __restrict__ Dd, float* __restrict__ dq_acc) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    constexpr int PER = D / 32;
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < PER; c += 2) {
        float2 a = unpack_bf16(*reinterpret_cast<const uint32_t*>(O + row * D + lane * PER + c));
        float2 b = unpack_bf16(*reinterpret_cast<const uint32_t*>(dO + row * D + lane * PER + c));
        s = fmaf(a.x, b.x, fmaf(a.y, b.y, s));
    }
    s = warp_sum(s);
    if (lane == 0) Dd[row] = s;
#pragma unroll
    for (int c = 0; c < PER; ++c) dq_acc[row * D + lane * PER + c] = 0.f;
}

__global__ void bwd_finalize_kernel(const float* __restrict__ dq_acc, int64_t n, float scale,
                                    __nv_bfloat16* __restrict__ dQ) {
    int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (e >= n) return;
    float4 v = *reinterpret_cast<const float4*>(dq_acc + e);
    *reinterpret_cast<uint2*>(dQ + e) = make_uint2(pack_bf16(v.x * scale, v.y * scale), pack_bf16(v.z * scale, v.w * scale));
}

// deterministic dQ: per query, sum its partials in (slot, slab) order.
template <int D>
__global__ void bwd_dq_combine_kernel(const float* __restrict__ dq_part, int64_t part_stride, int slabs,
                                      const int32_t* __restrict__ row_pos, int64_t N, int width, int64_t rows,
                                      float scale, __nv_bfloat16* __restrict__ dQ) {
    constexpr int PER = D / 32;
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const int64_t h = row / N;
    int32_t p = (lane < width) ? row_pos[row * width + lane] : -1;
    float acc[PER];
#pragma unroll
    for (int c = 0; c < PER; ++c) acc[c] = 0.f;
    for (int s = 0; s < width; ++s) {
        int32_t ps = __shfl_sync(0xffffffffu, p, s);
        if (ps < 0) continue;
        for (int sl = 0; sl < slabs; ++sl) {
            const float* src = dq_part + sl * part_stride + (h * N * width + ps) * D + lane * PER;
#pragma unroll
            for (int c = 0; c < PER; ++c) acc[c] += src[c];
        }
    }
    __nv_bfloat16* dst = dQ + row * D + lane * PER;
#pragma unroll
    for (int c = 0; c < PER; c += 2)
        *reinterpret_cast<uint32_t*>(dst + c) = pack_bf16(acc[c] * scale, acc[c + 1] * scale);
}

// workspace: Dd f32 [bh*N] | dq_acc f32 [bh*N*D] | (deterministic) dq_part
// f32 [slabs][bh*N*width*D]
static int bwd_kt(int B) { return B > 64 ? 128 : 64; }
static size_t bwd_ws(int64_t bh, int64_t N, int D, int B, int width, bool det) {
    size_t w = align_up((size_t)bh * N * 4, 256) + align_up((size_t)bh * N * D * 4, 256);
    if (det) w += (size_t)ceil_div(B, bwd_kt(B)) * bh * N * width * D * 4;
    return w;
}

template <int D, int KT>
static int launch_bwd_main(const void* q, const void* k, const void* v, const void* dout, const float* lse,
                           const float* Dd, int64_t bh, int64_t N, int B, int width, const int32_t* counts,
                           const int32_t* offsets, const int32_t* flat, float scale, float* dq_acc,
                           float* dq_part, int64_t part_stride, void* dk, void* dv, cudaStream_t s) {
    const int64_t n = ceil_div(N, B);
    const int slabs = (int)ceil_div(B, KT);
    const size_t smem = (size_t)2 * KT * D * 2 + 2 * kBwdBM * D * 2 + KT * 128 + kBwdBM * 12;
    auto kern = moba_bwd_mma_kernel<D, KT>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid((unsigned)(n * slabs), (unsigned)bh);
    kern<<<grid, KT * 2, smem, s>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k, (const __nv_bfloat16*)v,
                                    (const __nv_bfloat16*)dout, lse, Dd, N, B, width, counts, offsets, flat, scale,
                                    dq_acc, dq_part, part_stride, (__nv_bfloat16*)dk, (__nv_bfloat16*)dv);
    return check_launch("moba_bwd_mma_kernel");
}

template <int D>
static int launch_bwd(const void* q, const void* k, const void* v, const void* out, const void* dout,
                      const float* lse, int64_t bh, int64_t N, int B, int width, const int32_t* counts,
                      const int32_t* offsets, const int32_t* flat, const int32_t* row_pos, bool det, float scale,
                      void* dq, void* dk, void* dv, uint8_t* ws, cudaStream_t s) {
    float* Dd = (float*)ws;
    float* dq_acc = (float*)(ws + align_up((size_t)bh * N * 4, 256));
    float* dq_part = det ? (float*)((uint8_t*)dq_acc + align_up((size_t)bh * N * D * 4, 256)) : nullptr;
    const int64_t part_stride = bh * N * width * D;
    const int slabs = (int)ceil_div(B, bwd_kt(B));
    const int64_t rows = bh * N;
    {
    StageTimer tm(T_BWD_PRE, s);
    bwd_preprocess_kernel<D><<<(unsigned)ceil_div(rows, 8), 256, 0, s>>>((const __nv_bfloat16*)out,
                                                                        (const __nv_bfloat16*)dout, rows, Dd, dq_acc);
    }
    int st = check_launch("bwd_preprocess_kernel");
    if (st) return st;
    {
    StageTimer tm(T_BWD, s);
    if (B > 64)
        st = launch_bwd_main<D, 128>(q, k, v, dout, lse, Dd, bh, N, B, width, counts, offsets, flat, scale, dq_acc,
                                     dq_part, part_stride, dk, dv, s);
    else
        st = launch_bwd_main<D, 64>(q, k, v, dout, lse, Dd, bh, N, B, width, counts, offsets, flat, scale, dq_acc,
                                    dq_part, part_stride, dk, dv, s);
    }
    if (st) return st;
    StageTimer tm(T_BWD_POST, s);
    if (det) {
        bwd_dq_combine_kernel<D><<<(unsigned)ceil_div(rows, 8), 256, 0, s>>>(dq_part, part_stride, slabs, row_pos, N,
                                                                           width, rows, scale, (__nv_bfloat16*)dq);
        return check_launch("bwd_dq_combine_kernel");
    }
    const int64_t ne = rows * D;
    bwd_finalize_kernel<<<(unsigned)ceil_div(ne / 4, 256), 256, 0, s>>>(dq_acc, ne, scale, (__nv_bfloat16*)dq);
    return check_launch("bwd_finalize_kernel");
}

}  // namespace moba

using namespace moba;

extern "C" size_t moba_bwd_workspace_size(int64_t bh, int64_t n_tokens, int head_dim, int block_size, int width,
                                          int deterministic) {
    if (bh < 1 || n_tokens < 1 || block_size < 1 || width < 1) return 0;
    return bwd_ws(bh, n_tokens, head_dim, block_size, width, deterministic != 0);
}

extern "C" int moba_bwd(const void* q, const void* k, const void* v, const void* out, const void* dout,
                        const float* lse, int64_t bh, int64_t n_tokens, int head_dim, int block_size, int width,
                        const int32_t* counts, const int32_t* offsets, const int32_t* flat, const int32_t* row_pos,
                        int deterministic, float softmax_scale, void* dq, void* dk, void* dv, void* workspace,
                        size_t workspace_bytes, void* stream) {
    if (bh < 1 || bh > 65535 || n_tokens < 1 || block_size < 1 || width < 1) return MOBA_ERR_SHAPE;
    if (block_size > 256 || width > 32) return MOBA_ERR_UNSUPPORTED;
    const bool det = deterministic != 0;
    if (det && row_pos == nullptr) return MOBA_ERR_PLAN;
    if (workspace_bytes < bwd_ws(bh, n_tokens, head_dim, block_size, width, det)) return MOBA_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t* ws = (uint8_t*)workspace;
    if (head_dim == 64)
        return launch_bwd<64>(q, k, v, out, dout, lse, bh, n_tokens, block_size, width, counts, offsets, flat,
                              row_pos, det, softmax_scale, dq, dk, dv, ws, s);
    if (head_dim == 128)
        return launch_bwd<128>(q, k, v, out, dout, lse, bh, n_tokens, block_size, width, counts, offsets, flat,
                               row_pos, det, softmax_scale, dq, dk, dv, ws, s);
    return MOBA_ERR_UNSUPPORTED;
}
