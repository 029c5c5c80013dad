// Stage 1: key-block centroids, optionally fused with the causal key
// short-conv (src/router.py:32-46, src/keyconv.py:59-78).
//
// One CTA per (head, key block). HBM-bound: reads the block's K rows once
// (the width-1 halo rows above the block come from L2), writes K' (bf16)
// when the conv is on, and one fp32 centroid row.
#include "common.cuh"
#include <algorithm>
#include <type_traits>

namespace moba {

constexpr int kCentThreads = 256;
constexpr int kMaxConv = 5;

__device__ __forceinline__ float sigmoidf_acc(float x) {
    // overflow-safe two-branch form, as src/keyconv.py:50-56
    float e = expf(-fabsf(x));
    return x >= 0.f ? 1.f / (1.f + e) : e / (1.f + e);
}

__global__ void __launch_bounds__(kCentThreads)
centroid_conv_kernel(const __nv_bfloat16* __restrict__ K, const float* __restrict__ W, int width,
                     int64_t N, int D, int B, __nv_bfloat16* __restrict__ Kout,
                     float* __restrict__ cent) {
    extern __shared__ float red[];  // [row_groups][D]
    const int j = blockIdx.x;
    const int64_t h = blockIdx.y;
    const int n_blocks = (int)((N + B - 1) / B);
    const int CG = D / 8;                 // 16-byte column groups
    const int RG = kCentThreads / CG;     // row groups
    const int cg = threadIdx.x % CG;
    const int rg = threadIdx.x / CG;
    const int64_t t0 = (int64_t)j * B;
    const int len = (int)min64(B, N - t0);
    const __nv_bfloat16* Kh = K + h * N * D;

    float w[kMaxConv][8];
#pragma unroll
    for (int l = 0; l < kMaxConv; ++l)
#pragma unroll
        for (int c = 0; c < 8; ++c) w[l][c] = (l < width) ? W[l * D + cg * 8 + c] : 0.f;

    float acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = 0.f;

    for (int r = rg; r < len; r += RG) {
        const int64_t t = t0 + r;
        uint4 raw = *reinterpret_cast<const uint4*>(Kh + t * D + cg * 8);
        float x[8];
        {
            const uint32_t* u = reinterpret_cast<const uint32_t*>(&raw);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                float2 f = unpack_bf16(u[c]);
                x[2 * c] = f.x;
                x[2 * c + 1] = f.y;
            }
        }
        if (width > 0) {
            float a[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) a[c] = w[0][c] * x[c];
#pragma unroll
            for (int l = 1; l < kMaxConv; ++l) {
                if (l < width && t - l >= 0) {
                    uint4 rr = *reinterpret_cast<const uint4*>(Kh + (t - l) * D + cg * 8);
                    const uint32_t* u = reinterpret_cast<const uint32_t*>(&rr);
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        float2 f = unpack_bf16(u[c]);
                        a[2 * c] = fmaf(w[l][2 * c], f.x, a[2 * c]);
                        a[2 * c + 1] = fmaf(w[l][2 * c + 1], f.y, a[2 * c + 1]);
                    }
                }
            }
            uint32_t o[4];
#pragma unroll
            for (int c = 0; c < 8; ++c) x[c] = x[c] + a[c] * sigmoidf_acc(a[c]);
#pragma unroll
            for (int c = 0; c < 4; ++c) o[c] = pack_bf16(x[2 * c], x[2 * c + 1]);
            *reinterpret_cast<uint4*>(Kout + h * N * D + t * D + cg * 8) = make_uint4(o[0], o[1], o[2], o[3]);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] += x[c];
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) red[rg * D + cg * 8 + c] = acc[c];
    __syncthreads();
    for (int c = threadIdx.x; c < D; c += kCentThreads) {
        float s = 0.f;
        for (int g = 0; g < RG; ++g) s += red[g * D + c];
        cent[(h * n_blocks + j) * D + c] = s / (float)len;
    }
}

// Plain centroids (no conv): one 4-warp CTA per (head, block). L = D/8
// lanes cover a 16-B-per-lane row, each warp takes every 4th group of 32/L
// rows with all of its loads in flight before any is summed, lane groups
// are folded with shuffles and the 4 warps through shared memory. The
// per-column summation order is fixed (deterministic).
template <int D, typename KT>
__global__ void __launch_bounds__(128)
centroid_warp_kernel(const KT* __restrict__ K, int64_t N, int B, int64_t total_blocks,
                     float* __restrict__ cent) {
    constexpr int L = D / 8, G = 32 / L, U = 8, W = 4;
    __shared__ float part[W][D];
    const int64_t wb = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, grp = lane / L, sub = lane % L;
    const int n_blocks = (int)((N + B - 1) / B);
    const int64_t h = wb / n_blocks;
    const int j = (int)(wb - h * n_blocks);
    const int64_t t0 = (int64_t)j * B;
    const int len = (int)min64(B, N - t0);
    const KT* base = K + (h * N + t0) * D + sub * 8;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int r0 = warp * G + grp; r0 < len; r0 += U * W * G) {
        float x[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int r = r0 + u * W * G;
            if (r < len) {
                ld8f(base + (int64_t)r * D, x[u]);
            } else {
#pragma unroll
                for (int c = 0; c < 8; ++c) x[u][c] = 0.f;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[c] += x[u][c];
    }
#pragma unroll
    for (int o = L; o < 32; o <<= 1)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
    if (grp == 0)
#pragma unroll
        for (int c = 0; c < 8; ++c) part[warp][sub * 8 + c] = acc[c];
    __syncthreads();
    if (threadIdx.x < D) {
        const float sum = (part[0][threadIdx.x] + part[1][threadIdx.x]) + (part[2][threadIdx.x] + part[3][threadIdx.x]);
        cent[wb * D + threadIdx.x] = sum / (float)len;
    }
}

// Conv + centroids, vectorised (D in {64, 128}): one 128-thread CTA per
// (head, block); a thread handles 8 channels of a row with 16-B loads of K
// and its width-1 predecessors (L1 hits), writes K' (bf16) and accumulates
// the unrounded fp32 K' for the centroid; fixed-order reduction.
template <int D, int width, typename KT>
__global__ void __launch_bounds__(128)
centroid_conv_vec_kernel(const KT* __restrict__ K, const float* __restrict__ W, int64_t N, int B,
                         __nv_bfloat16* __restrict__ Kout, float* __restrict__ cent) {
    constexpr int G = D / 8, RS = 128 / G;
    __shared__ float red[RS][D];
    const int j = blockIdx.x;
    const int64_t h = blockIdx.y;
    const int n_blocks = (int)((N + B - 1) / B);
    const int grp = threadIdx.x % G, rs = threadIdx.x / G;
    const int64_t t0 = (int64_t)j * B;
    const int len = (int)min64(B, N - t0);
    const KT* Kh = K + h * N * D + grp * 8;
    uint4* Ko = reinterpret_cast<uint4*>(Kout + h * N * D);
    float w[width][8];
#pragma unroll
    for (int l = 0; l < width; ++l)
#pragma unroll
        for (int c = 0; c < 8; ++c) w[l][c] = W[l * D + grp * 8 + c];
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int r = rs; r < len; r += RS) {
        const int64_t t = t0 + r;
        float xs[width][8];
#pragma unroll
        for (int l = 0; l < width; ++l) {
            if (t - l >= 0) {
                ld8f(Kh + (t - l) * D, xs[l]);
            } else {
#pragma unroll
                for (int c = 0; c < 8; ++c) xs[l][c] = 0.f;
            }
        }
        float x[8], a[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            x[c] = xs[0][c];
            a[c] = w[0][c] * xs[0][c];
        }
#pragma unroll
        for (int l = 1; l < width; ++l)
#pragma unroll
            for (int c = 0; c < 8; ++c) a[c] = fmaf(w[l][c], xs[l][c], a[c]);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            x[c] = x[c] + a[c] * sigmoidf_acc(a[c]);      // K' = K + silu(conv(K)) (src/keyconv.py:77-78)
            acc[c] += x[c];
        }
        Ko[t * G + grp] = make_uint4(pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]), pack_bf16(x[4], x[5]),
                                     pack_bf16(x[6], x[7]));
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) red[rs][grp * 8 + c] = acc[c];
    __syncthreads();
    if (threadIdx.x < D) {
        float sum = 0.f;
        for (int g2 = 0; g2 < RS; ++g2) sum += red[g2][threadIdx.x];
        cent[(h * n_blocks + j) * D + threadIdx.x] = sum / (float)len;
    }
}

// ---------------------------------------------------------------- conv backward
// key_conv_backward (src/keyconv.py:81-104). One CTA per (head, 64-row
// chunk): g over the chunk plus a (width-1)-row lookahead in smem, then
// dK_t = dK'_t + sum_l W[l] g_{t+l}; per-CTA dW partials reduced by a
// second kernel (deterministic, no atomics).
constexpr int kConvRows = 64;

__global__ void __launch_bounds__(256)
conv_bwd_kernel(const __nv_bfloat16* __restrict__ K, const float* __restrict__ W, int width,
                const __nv_bfloat16* __restrict__ dKc, int64_t N, int D,
                __nv_bfloat16* __restrict__ dK, float* __restrict__ dw_part) {
    extern __shared__ float g_s[];  // [(kConvRows + kMaxConv - 1)][D]
    const int64_t h = blockIdx.y;
    const int64_t t0 = (int64_t)blockIdx.x * kConvRows;
    const __nv_bfloat16* Kh = K + h * N * D;
    const __nv_bfloat16* dKch = dKc + h * N * D;
    const int rows = kConvRows + width - 1;
    for (int e = threadIdx.x; e < rows * D; e += blockDim.x) {
        int r = e / D, c = e % D;
        int64_t t = t0 + r;
        float g = 0.f;
        if (t < N) {
            float a = 0.f;
            for (int l = 0; l < width; ++l)
                if (t - l >= 0) a = fmaf(W[l * D + c], __bfloat162float(Kh[(t - l) * D + c]), a);
            float s = sigmoidf_acc(a);
            g = __bfloat162float(dKch[t * D + c]) * (s * (1.f + a * (1.f - s)));
        }
        g_s[r * D + c] = g;
    }
    __syncthreads();
    // dK and dW partials: thread (row group rg, channel c) handles rows rg, rg+RG, ...
    float* red = g_s + rows * D;  // [RG][kMaxConv][D] partial dW
    const int RG = blockDim.x / D;
    const int c = threadIdx.x % D, rg = threadIdx.x / D;
    float dwl[kMaxConv] = {0.f, 0.f, 0.f, 0.f, 0.f};
    float wl[kMaxConv];
    for (int l = 0; l < kMaxConv; ++l) wl[l] = (l < width) ? W[l * D + c] : 0.f;
    for (int r = rg; r < kConvRows; r += RG) {
        const int64_t t = t0 + r;
        if (t >= N) break;
        float v = __bfloat162float(dKch[t * D + c]);
        for (int l = 0; l < width; ++l) v = fmaf(wl[l], g_s[(r + l) * D + c], v);
        dK[h * N * D + t * D + c] = __float2bfloat16(v);
        const float gt = g_s[r * D + c];
        for (int l = 0; l < width; ++l)
            if (t - l >= 0) dwl[l] = fmaf(gt, __bfloat162float(Kh[(t - l) * D + c]), dwl[l]);
    }
    for (int l = 0; l < width; ++l) red[(rg * kMaxConv + l) * D + c] = dwl[l];
    __syncthreads();
    if (rg == 0) {
        const int64_t part = h * gridDim.x + blockIdx.x;
        for (int l = 0; l < width; ++l) {
            float acc = 0.f;
            for (int gI = 0; gI < RG; ++gI) acc += red[(gI * kMaxConv + l) * D + c];
            dw_part[(part * width + l) * D + c] = acc;
        }
    }
}

// Vectorised conv backward (D in {64, 128}): one CTA per (head, 64-row
// chunk), 8 channels per thread with 16-B loads. K rows (with a width-1
// halo on both sides) and dK' rows are staged in shared memory once; g, dK
// and the per-CTA dW partials (fixed-order warp + CTA reductions) follow.
template <int D, int width>
__global__ void __launch_bounds__(256)
conv_bwd_vec_kernel(const __nv_bfloat16* __restrict__ K, const float* __restrict__ W,
                    const __nv_bfloat16* __restrict__ dKc, int64_t N, __nv_bfloat16* __restrict__ dK,
                    float* __restrict__ dw_part) {
    constexpr int G = D / 8;                    // 8-channel groups
    constexpr int RS = 256 / G;                 // row slots
    constexpr int RK = kConvRows + 2 * (kMaxConv - 1);
    constexpr int RG = kConvRows + kMaxConv - 1;
    extern __shared__ __align__(16) uint8_t cb_smem[];
    uint4* Ks = reinterpret_cast<uint4*>(cb_smem);                       // [RK][G] bf16x8
    uint4* dks = Ks + RK * G;                                            // [RG][G] bf16x8
    float4* gs = reinterpret_cast<float4*>(dks + RG * G);                // [RG][G][2] fp32x8
    float* red = reinterpret_cast<float*>(gs + RG * G * 2);              // [8 warps][kMaxConv][D]
    const int64_t h = blockIdx.y;
    const int64_t t0 = (int64_t)blockIdx.x * kConvRows;
    const int tid = threadIdx.x, grp = tid % G, rs = tid / G;
    const int halo = width - 1;
    const uint4* Kh = reinterpret_cast<const uint4*>(K + h * N * D);
    const uint4* dKh = reinterpret_cast<const uint4*>(dKc + h * N * D);
    // stage K rows [t0 - halo, t0 + 64 + halo) and dK' rows [t0, t0 + 64 + halo)
    for (int e = tid; e < (kConvRows + 2 * halo) * G; e += 256) {
        const int r = e / G, c = e % G;
        const int64_t t = t0 - halo + r;
        Ks[r * G + c] = (t >= 0 && t < N) ? __ldg(Kh + t * G + c) : make_uint4(0, 0, 0, 0);
    }
    for (int e = tid; e < (kConvRows + halo) * G; e += 256) {
        const int r = e / G, c = e % G;
        const int64_t t = t0 + r;
        dks[r * G + c] = (t < N) ? __ldg(dKh + t * G + c) : make_uint4(0, 0, 0, 0);
    }
    float w[width][8];
#pragma unroll
    for (int l = 0; l < width; ++l)
#pragma unroll
        for (int c = 0; c < 8; ++c) w[l][c] = W[l * D + grp * 8 + c];
    __syncthreads();
    auto unpack8 = [](uint4 u, float (&x)[8]) {
        const uint32_t v[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const float2 f = unpack_bf16(v[c]);
            x[2 * c] = f.x;
            x[2 * c + 1] = f.y;
        }
    };
    // g_t = dK'_t * silu'(a_t), a_t = sum_l W[l] K[t-l] (src/keyconv.py:96)
    for (int r = rs; r < kConvRows + halo; r += RS) {
        const int64_t t = t0 + r;
        float g[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (t < N) {
            float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
            for (int l = 0; l < width; ++l) {
                float x[8];
                unpack8(Ks[(r + halo - l) * G + grp], x);
#pragma unroll
                for (int c = 0; c < 8; ++c) a[c] = fmaf(w[l][c], x[c], a[c]);
            }
            float dk[8];
            unpack8(dks[r * G + grp], dk);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const float sg = sigmoidf_acc(a[c]);
                g[c] = dk[c] * (sg * (1.f + a[c] * (1.f - sg)));
            }
        }
        gs[(r * G + grp) * 2] = make_float4(g[0], g[1], g[2], g[3]);
        gs[(r * G + grp) * 2 + 1] = make_float4(g[4], g[5], g[6], g[7]);
    }
    __syncthreads();
    // dK_t = dK'_t + sum_l W[l] g_{t+l};  dW[l] += g_t K_{t-l}  (src/keyconv.py:97-103)
    float dwl[width][8];
#pragma unroll
    for (int l = 0; l < width; ++l)
#pragma unroll
        for (int c = 0; c < 8; ++c) dwl[l][c] = 0.f;
    uint4* dKo = reinterpret_cast<uint4*>(dK + h * N * D);
    for (int r = rs; r < kConvRows; r += RS) {
        const int64_t t = t0 + r;
        if (t >= N) break;
        float v[8];
        unpack8(dks[r * G + grp], v);
        float gt[8];
        {
            const float4 a = gs[(r * G + grp) * 2], b = gs[(r * G + grp) * 2 + 1];
            gt[0] = a.x; gt[1] = a.y; gt[2] = a.z; gt[3] = a.w; gt[4] = b.x; gt[5] = b.y; gt[6] = b.z; gt[7] = b.w;
        }
#pragma unroll
        for (int l = 0; l < width; ++l) {
            const float4 a = gs[((r + l) * G + grp) * 2], b = gs[((r + l) * G + grp) * 2 + 1];
            const float gl[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
            float x[8];
            unpack8(Ks[(r + halo - l) * G + grp], x);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                v[c] = fmaf(w[l][c], gl[c], v[c]);
                dwl[l][c] = fmaf(gt[c], x[c], dwl[l][c]);
            }
        }
        dKo[t * G + grp] = make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
                                      pack_bf16(v[6], v[7]));
    }
    // dW partial: lanes of a warp with the same channel group (xor over the
    // row-slot bits), then the 8 warps in order
#pragma unroll
    for (int l = 0; l < width; ++l)
#pragma unroll
        for (int c = 0; c < 8; ++c)
#pragma unroll
            for (int o = G; o < 32; o <<= 1) dwl[l][c] += __shfl_xor_sync(0xffffffffu, dwl[l][c], o);
    const int warp = tid >> 5, lane = tid & 31;
    if (lane < G) {
#pragma unroll
        for (int l = 0; l < width; ++l)
#pragma unroll
            for (int c = 0; c < 8; ++c) red[(warp * kMaxConv + l) * D + lane * 8 + c] = dwl[l][c];
    }
    __syncthreads();
    const int64_t part = h * gridDim.x + blockIdx.x;
    for (int e = tid; e < width * D; e += 256) {
        const int l = e / D, c = e % D;
        float acc = 0.f;
        for (int wp = 0; wp < 8; ++wp) acc += red[(wp * kMaxConv + l) * D + c];
        dw_part[(part * width + l) * D + c] = acc;
    }
}

__global__ void conv_dw_reduce_kernel(const float* __restrict__ dw_part, int64_t n_parts, int width, int D,
                                      float* __restrict__ dw) {
    // one CTA per dW element, fixed-order strided sums + tree (deterministic)
    __shared__ float red[256];
    const int e = blockIdx.x;
    float s = 0.f;
    for (int64_t p = threadIdx.x; p < n_parts; p += blockDim.x) s += dw_part[p * width * D + e];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) dw[e] = red[0];
}

template <typename KT>
static int run_centroids(const KT* k, const float* conv_w, int conv_width, int64_t bh, int64_t n_tokens,
                         int head_dim, int block_size, void* k_conv_out, float* centroids, cudaStream_t s) {
    if (bh < 1 || n_tokens < 1 || block_size < 1) return MOBA_ERR_SHAPE;
    if (head_dim % 8 != 0 || head_dim > 256) return MOBA_ERR_UNSUPPORTED;
    if (conv_width < 0 || conv_width > kMaxConv) return MOBA_ERR_CONFIG;
    if (conv_width > 0 && (conv_w == nullptr || k_conv_out == nullptr)) return MOBA_ERR_CONFIG;
    const int64_t n_blocks = ceil_div(n_tokens, block_size);
    if (n_blocks > 2147483647 || bh > 65535) return MOBA_ERR_UNSUPPORTED;
    StageTimer tm(T_CENTROID, s);
    if (conv_width == 0 && (head_dim == 64 || head_dim == 128)) {
        const int64_t total = bh * n_blocks;
        if (head_dim == 64)
            centroid_warp_kernel<64, KT><<<(unsigned)total, 128, 0, s>>>(k, n_tokens, block_size, total, centroids);
        else
            centroid_warp_kernel<128, KT><<<(unsigned)total, 128, 0, s>>>(k, n_tokens, block_size, total, centroids);
        return check_launch("centroid_warp_kernel");
    }
    if (head_dim == 64 || head_dim == 128) {
        using KernT = void (*)(const KT*, const float*, int64_t, int, __nv_bfloat16*, float*);
        static const KernT k64[kMaxConv] = {centroid_conv_vec_kernel<64, 1, KT>, centroid_conv_vec_kernel<64, 2, KT>,
                                            centroid_conv_vec_kernel<64, 3, KT>, centroid_conv_vec_kernel<64, 4, KT>,
                                            centroid_conv_vec_kernel<64, 5, KT>};
        static const KernT k128[kMaxConv] = {centroid_conv_vec_kernel<128, 1, KT>, centroid_conv_vec_kernel<128, 2, KT>,
                                             centroid_conv_vec_kernel<128, 3, KT>, centroid_conv_vec_kernel<128, 4, KT>,
                                             centroid_conv_vec_kernel<128, 5, KT>};
        const KernT kern = head_dim == 64 ? k64[conv_width - 1] : k128[conv_width - 1];
        kern<<<dim3((unsigned)n_blocks, (unsigned)bh), 128, 0, s>>>(k, conv_w, n_tokens, block_size,
                                                                   (__nv_bfloat16*)k_conv_out, centroids);
        return check_launch("centroid_conv_vec_kernel");
    }
    if constexpr (std::is_same<KT, __nv_bfloat16>::value) {
        const int RG = kCentThreads / (head_dim / 8);
        const size_t smem = (size_t)RG * head_dim * sizeof(float);
        centroid_conv_kernel<<<dim3((unsigned)n_blocks, (unsigned)bh), kCentThreads, smem, s>>>(
            k, conv_w, conv_width, n_tokens, head_dim, block_size, (__nv_bfloat16*)k_conv_out, centroids);
        return check_launch("centroid_conv_kernel");
    }
    return MOBA_ERR_UNSUPPORTED;
}

}  // namespace moba

using namespace moba;

extern "C" int moba_centroids(const void* k, const float* conv_w, int conv_width, int64_t bh,
                              int64_t n_tokens, int head_dim, int block_size, void* k_conv_out,
                              float* centroids, void* stream) {
    clear_last_error();
    return run_centroids((const __nv_bfloat16*)k, conv_w, conv_width, bh, n_tokens, head_dim, block_size, k_conv_out,
                         centroids, (cudaStream_t)stream);
}

extern "C" int moba_centroids_f32(const float* k, const float* conv_w, int conv_width, int64_t bh,
                                  int64_t n_tokens, int head_dim, int block_size, void* k_conv_out,
                                  float* centroids, void* stream) {
    clear_last_error();
    return run_centroids(k, conv_w, conv_width, bh, n_tokens, head_dim, block_size, k_conv_out, centroids,
                         (cudaStream_t)stream);
}

extern "C" size_t moba_conv_bwd_workspace_size(int64_t bh, int64_t n_tokens, int head_dim, int conv_width) {
    return (size_t)bh * ceil_div(n_tokens, kConvRows) * conv_width * head_dim * sizeof(float);
}

extern "C" int moba_conv_bwd(const void* k, const float* conv_w, int conv_width, const void* dk_conv,
                             int64_t bh, int64_t n_tokens, int head_dim, void* dk, float* dw,
                             void* workspace, size_t workspace_bytes, void* stream) {
    clear_last_error();
    if (bh < 1 || n_tokens < 1 || head_dim < 1) return MOBA_ERR_SHAPE;
    if (conv_width < 1 || conv_width > kMaxConv) return MOBA_ERR_CONFIG;
    if (workspace_bytes < moba_conv_bwd_workspace_size(bh, n_tokens, head_dim, conv_width))
        return MOBA_ERR_WORKSPACE;
    dim3 grid((unsigned)ceil_div(n_tokens, kConvRows), (unsigned)bh);
    const int threads = std::max(head_dim, (256 / head_dim) * head_dim);
    size_t smem = (size_t)(kConvRows + conv_width - 1) * head_dim * sizeof(float) +
                  (size_t)(threads / head_dim) * kMaxConv * head_dim * sizeof(float);
    if (smem > 48 * 1024) {
        cudaFuncSetAttribute(conv_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    cudaStream_t s = (cudaStream_t)stream;
    StageTimer tm(T_CONV_BWD, s);
    if (head_dim == 64 || head_dim == 128) {
        const int G = head_dim / 8;
        const size_t vsmem = (size_t)(kConvRows + 2 * (kMaxConv - 1)) * G * 16 + (size_t)(kConvRows + kMaxConv - 1) * G * 16 +
                             (size_t)(kConvRows + kMaxConv - 1) * G * 32 + (size_t)8 * kMaxConv * head_dim * 4;
        using KernT = void (*)(const __nv_bfloat16*, const float*, const __nv_bfloat16*, int64_t, __nv_bfloat16*,
                               float*);
        static const KernT k64[kMaxConv] = {conv_bwd_vec_kernel<64, 1>, conv_bwd_vec_kernel<64, 2>,
                                            conv_bwd_vec_kernel<64, 3>, conv_bwd_vec_kernel<64, 4>,
                                            conv_bwd_vec_kernel<64, 5>};
        static const KernT k128[kMaxConv] = {conv_bwd_vec_kernel<128, 1>, conv_bwd_vec_kernel<128, 2>,
                                             conv_bwd_vec_kernel<128, 3>, conv_bwd_vec_kernel<128, 4>,
                                             conv_bwd_vec_kernel<128, 5>};
        const KernT kern = head_dim == 64 ? k64[conv_width - 1] : k128[conv_width - 1];
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vsmem);
        kern<<<grid, 256, vsmem, s>>>((const __nv_bfloat16*)k, conv_w, (const __nv_bfloat16*)dk_conv, n_tokens,
                                      (__nv_bfloat16*)dk, (float*)workspace);
    } else {
        conv_bwd_kernel<<<grid, threads, smem, s>>>((const __nv_bfloat16*)k, conv_w, conv_width,
                                                (const __nv_bfloat16*)dk_conv, n_tokens, head_dim,
                                                (__nv_bfloat16*)dk, (float*)workspace);
    }
    int st = check_launch("conv_bwd_kernel");
    if (st) return st;
    int e = conv_width * head_dim;
    conv_dw_reduce_kernel<<<e, 256, 0, s>>>((const float*)workspace, bh * grid.x,
                                                           conv_width, head_dim, dw);
    return check_launch("conv_dw_reduce_kernel");
}
