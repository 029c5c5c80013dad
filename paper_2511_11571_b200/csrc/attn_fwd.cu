// Forward host side + combine (moba_forward, src/attention.py:147-182;
// paper Alg. 1), key-block-major.
//
// Work item = (head, key block j, 128-row tile of block j's varlen slice,
// 128-key slab of the block). The tcgen05 kernel in attn_fwd_ts.cu gathers
// the tile's query rows (flat_queries), streams K_j / V_j, and writes one
// partial per (query, block, slab): O_s normalised (bf16) and lse_s (fp32) at
// the pair's flat position. moba_combine merges a query's partials into O
// and LSE (SoftmaxState.finalize over the query's blocks,
// src/attention.py:70-74).
#include "common.cuh"
#include "sm100.cuh"

namespace moba {

constexpr int kTileM = 128;       // gathered query rows per item
constexpr float kLog2e = 1.4426950408889634f;

// ---------------------------------------------------------------- combine
// L = D/8 lanes per query (16 B of a partial row each), so a warp merges
// 32/L queries at once (4 at d = 64, 2 at d = 128) with no cross-lane
// reduction of the output: lane `sub` of a group owns elements
// [8 sub, 8 sub + 8) of its query's row. Virtual slot v = slot * slabs + slab
// lives at partial position row_pos[slot] * slabs + slab; the group's lanes
// load the positions and LSEs of slots sub, sub + L, ... and broadcast them
// with in-group shuffles. Every partial row of a batch of up to 16 slots is
// requested before any is consumed. (The former one-query-per-warp layout
// issued ~460 instructions per query and was issue bound: ncu 83% issue
// active at N = 64K.)
template <int D, int VW, bool kOneSlab>
__global__ void __launch_bounds__(128)
moba_combine_kernel(const __nv_bfloat16* __restrict__ part_o, const float* __restrict__ part_lse,
                    const int32_t* __restrict__ row_pos, int64_t N, int width, int slabs, int64_t total_rows,
                    __nv_bfloat16* __restrict__ O, float* __restrict__ LSE) {
    constexpr int L = D / 8;                 // lanes per query
    constexpr int QPW = 32 / L;              // queries per warp
    constexpr int C = (VW + L - 1) / L;      // slot chunks per lane
    constexpr int NB = VW < 16 ? VW : 16;    // partial rows in flight per lane
    const int vwidth = kOneSlab ? width : width * slabs;
    const int lane = threadIdx.x & 31, grp = lane / L, sub = lane % L, g0 = grp * L;
    const int64_t row = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * QPW + grp;
    const bool ok = row < total_rows;
    const int64_t r = ok ? row : total_rows - 1;
    const int64_t h = total_rows < (1ll << 31) ? (int64_t)((uint32_t)r / (uint32_t)N) : r / N;
    const float* lse_h = part_lse + h * N * vwidth;
    int32_t p[C];
    float ls[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int v = sub + L * c;
        const int32_t q = (v < vwidth) ? __ldg(row_pos + r * width + (kOneSlab ? v : v / slabs)) : -1;
        p[c] = q >= 0 ? (kOneSlab ? q : q * slabs + v % slabs) : -1;
        ls[c] = (p[c] >= 0) ? __ldg(lse_h + p[c]) : -INFINITY;
    }
    float m = ls[0];
#pragma unroll
    for (int c = 1; c < C; ++c) m = fmaxf(m, ls[c]);
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float w[C], ws = 0.f;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        w[c] = (p[c] >= 0) ? __expf(ls[c] - m) : 0.f;
        ws += w[c];
    }
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) ws += __shfl_xor_sync(0xffffffffu, ws, o);
    const uint4* base = reinterpret_cast<const uint4*>(part_o + h * N * vwidth * D) + sub;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#pragma unroll
    for (int v0 = 0; v0 < VW; v0 += NB) {
        if (v0 >= vwidth) break;
        uint4 raw[NB];
        float wt[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const int v = v0 + u;            // compile-time: chunk v / L, held by lane g0 + v % L
            const int32_t pv = __shfl_sync(0xffffffffu, p[v / L], g0 + v % L);
            const float wv = __shfl_sync(0xffffffffu, w[v / L], g0 + v % L);
            const bool live = v < vwidth && pv >= 0;
            wt[u] = live ? wv : 0.f;
            raw[u] = live ? __ldg(base + (int64_t)pv * L) : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const uint32_t uu[4] = {raw[u].x, raw[u].y, raw[u].z, raw[u].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f = unpack_bf16(uu[e]);
                acc[2 * e] = fmaf(wt[u], f.x, acc[2 * e]);
                acc[2 * e + 1] = fmaf(wt[u], f.y, acc[2 * e + 1]);
            }
        }
    }
    if (!ok) return;
    const float inv = 1.f / ws;
    *(reinterpret_cast<uint4*>(O + row * D) + sub) =
        make_uint4(pack_bf16(acc[0] * inv, acc[1] * inv), pack_bf16(acc[2] * inv, acc[3] * inv),
                   pack_bf16(acc[4] * inv, acc[5] * inv), pack_bf16(acc[6] * inv, acc[7] * inv));
    if (sub == 0) LSE[row] = m + __logf(ws);
}

template <int D>
static void launch_combine(const void* part_o, const float* part_lse, const int32_t* row_pos, int64_t N, int width,
                           int S, int64_t rows, void* out, float* lse, cudaStream_t s) {
    // 4 warps x (32 / (D / 8)) queries per CTA (128-thread CTAs measured
    // faster than 256: 64K combine 0.57 -> 0.48 ms)
    const unsigned grid = (unsigned)ceil_div(rows, 4 * (256 / D));
    auto po = (const __nv_bfloat16*)part_o;
    auto o = (__nv_bfloat16*)out;
    const int vw = width * S;
#define MOBA_COMBINE(W)                                                                                    \
    (S == 1 ? moba_combine_kernel<D, W, true><<<grid, 128, 0, s>>>(po, part_lse, row_pos, N, width, S, rows, o, lse) \
            : moba_combine_kernel<D, W, false><<<grid, 128, 0, s>>>(po, part_lse, row_pos, N, width, S, rows, o, lse))
    // exact slot counts for the common widths (top-k 8 / 16 -> 9 / 17 slots)
    if (vw <= 4) MOBA_COMBINE(4);
    else if (vw <= 8) MOBA_COMBINE(8);
    else if (vw <= 9) MOBA_COMBINE(9);
    else if (vw <= 12) MOBA_COMBINE(12);
    else if (vw <= 16) MOBA_COMBINE(16);
    else if (vw <= 17) MOBA_COMBINE(17);
    else if (vw <= 24) MOBA_COMBINE(24);
    else if (vw <= 32) MOBA_COMBINE(32);
    else if (vw <= 64) MOBA_COMBINE(64);
    else MOBA_COMBINE(128);
#undef MOBA_COMBINE
}

// ---------------------------------------------------------------- work items
// One thread per (head, block): exclusive scan of item counts (128-row tiles
// x slabs) in a single CTA; fwd_ts_fill_items then writes each (head,
// block)'s item records at its offset.
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

size_t fwd_ts_item_bytes();

// workspace layout (all head-local regions back to back):
//   part_o   bf16 [bh, N*width*slabs, D]
//   part_lse f32  [bh, N*width*slabs]
//   item_off i32  [bh*n]
//   n_items  i32
//   items    Item [bh*(ceil(N*width/128) + n) * slabs]
struct FwdWs {
    size_t part_o, part_lse, item_off, n_items, items, total;
};

// blocks longer than 128 keys are processed as ceil(B / 128) slabs, each
// with its own partial
static int fwd_slabs(int B) { return (int)ceil_div(B, kTileM); }

static FwdWs fwd_ws_layout(int64_t bh, int64_t N, int D, int B, int width) {
    FwdWs w;
    const int64_t n = ceil_div(N, B);
    const int S = fwd_slabs(B);
    const int64_t E = N * width * S;
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
    off = align_up(off + (size_t)bh * (ceil_div(N * width, kTileM) + n) * S * fwd_ts_item_bytes(), 256);
    w.total = off;
    return w;
}

template <int D>
int launch_fwd_ts(const void* q, const void* k, const void* v, int64_t bh, int kv_group, int64_t N, int B, int width,
                  const int32_t* flat, const void* items, const int32_t* item_lo, const int32_t* item_hi,
                  float scale_log2, void* part_o, float* part_lse, cudaStream_t s);
void fwd_ts_fill_items(const int32_t* counts, const int32_t* offsets, const int32_t* item_off, int64_t total,
                       int slabs, void* items, cudaStream_t s);

template <int D>
static int launch_fwd(const void* q, const void* k, const void* v, int64_t bh, int kv_group, int64_t N, int B,
                      int width, const int32_t* counts, const int32_t* offsets, const int32_t* flat,
                      const int32_t* row_pos, float scale, void* out, float* lse, uint8_t* ws, const FwdWs& L,
                      cudaStream_t s) {
    const int64_t n = ceil_div(N, B);
    const int64_t total = bh * n;
    const int S = fwd_slabs(B);
    int32_t* item_off = (int32_t*)(ws + L.item_off);
    int32_t* n_items = (int32_t*)(ws + L.n_items);
    fwd_items_scan_kernel<<<1, 1024, 0, s>>>(counts, total, kTileM, S, item_off, n_items);
    int st = check_launch("fwd_items_scan_kernel");
    if (st) return st;
    fwd_ts_fill_items(counts, offsets, item_off, total, S, ws + L.items, s);
    st = check_launch("fwd_ts_items_kernel");
    if (st) return st;
    st = launch_fwd_ts<D>(q, k, v, bh, kv_group, N, B, width, flat, ws + L.items, item_off, n_items,
                          scale * kLog2e, ws + L.part_o, (float*)(ws + L.part_lse), s);
    if (st) return st;
    StageTimer tm(T_COMBINE, s);
    launch_combine<D>(ws + L.part_o, (const float*)(ws + L.part_lse), row_pos, N, width, S, bh * N, out, lse, s);
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
    clear_last_error();
    if (bh < 1 || n_tokens < 1 || block_size < 1 || width < 1) return MOBA_ERR_SHAPE;
    if (kv_group < 1 || bh % kv_group != 0) return MOBA_ERR_SHAPE;
    if (width > 32 || block_size > 512) return MOBA_ERR_UNSUPPORTED;
    if (n_tokens * width * fwd_slabs(block_size) >= (1ll << 31)) return MOBA_ERR_UNSUPPORTED;
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
