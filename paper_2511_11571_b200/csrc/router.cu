// Stages 2+3: tiled top-k routing and the key-block-major varlen plan.
//
//   select_topk  (src/router.py:49-120)   -> route_topk_fp32_kernel (parity mode),
//                                            route_tc_kernel (route_tc.cu, tensor cores)
//   build_varlen (src/router.py:123-154)  -> varlen_count / varlen_scan /
//                                            varlen_scatter kernels
//   validate_plan (src/core.py:254-296)   -> validate_* kernels
//
// The router never materialises the [N, n] score matrix: a CTA holds 128
// queries, streams 32-centroid chunks through shared memory, computes a
// 128x32 fp32 score tile with register-blocked FFMA (exact fp32 products of
// bf16 queries and fp32 centroids, summed in d order), and each thread keeps
// its query's running top-k list in registers.
#include "common.cuh"
#include "sm100.cuh"
#include <cstdlib>

namespace moba {

constexpr int kRouteQ = 128;    // queries per CTA (one per thread in selection)
constexpr int kRouteC = 32;     // centroids per chunk
constexpr int kRouteThreads = 128;

// Insert candidate (s, j) into a list sorted by (score desc, index asc).
// Candidates arrive in ascending j, so a tie with an existing entry keeps
// the existing (lower-index) entry first: ties -> lower block index
// (src/router.py:95-98). The displaced entries bubble down with the same
// (score, index) order so equal scores stay index-ordered.
template <int KMAX>
MOBA_DEV void topk_insert(float (&ts)[KMAX], int (&ti)[KMAX], float s, int j) {
    float cs = s;
    int ci = j;
#pragma unroll
    for (int u = 0; u < KMAX; ++u) {
        bool sw = (cs > ts[u]) || (cs == ts[u] && ci < ti[u]);
        float t = ts[u];
        int tt = ti[u];
        ts[u] = sw ? cs : t;
        ti[u] = sw ? ci : tt;
        cs = sw ? t : cs;
        ci = sw ? tt : ci;
    }
}


// Insert a candidate whose block index is larger than every listed one (a
// thread sees its candidates in ascending block order): it goes after every
// entry with score >= s (equal scores keep the lower index first,
// src/router.py:95-98). All slot tests read the old list, so the eight
// compare/select groups are independent; s = -inf is a no-op.
template <int KMAX>
MOBA_DEV void topk_insert_tail(float (&ts)[KMAX], int (&ti)[KMAX], float s, int j) {
    bool ge[KMAX];
#pragma unroll
    for (int u = 0; u < KMAX; ++u) ge[u] = ts[u] >= s;
#pragma unroll
    for (int u = KMAX - 1; u >= 1; --u) {
        const float ns = ge[u - 1] ? s : ts[u - 1];
        const int ni = ge[u - 1] ? j : ti[u - 1];
        ts[u] = ge[u] ? ts[u] : ns;
        ti[u] = ge[u] ? ti[u] : ni;
    }
    ts[0] = ge[0] ? ts[0] : s;
    ti[0] = ge[0] ? ti[0] : j;
}

// Chunked, warp-friendly selection: each lane first compacts the candidates
// of a 32-wide chunk that beat its (stale) threshold into a private smem
// list with predicated stores, then the warp inserts them in lockstep. The
// insert loop runs max-over-lanes(passes) times instead of once for every
// candidate any lane accepts. Candidates stay in ascending block order, so
// the (score desc, index asc) order of topk_insert is preserved.
template <int KMAX>
MOBA_DEV void select_chunk32(const float (&sv)[32], int j0, int lim, float (&ts)[KMAX], int (&ti)[KMAX],
                             float* buf_s, int* buf_i) {
    const float thr = ts[KMAX - 1];
    int cnt = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        if (i < lim && sv[i] > thr) {
            buf_s[cnt * 33] = sv[i];
            buf_i[cnt * 33] = j0 + i;
            ++cnt;
        }
    }
    const int iters = __reduce_max_sync(0xffffffffu, (unsigned)cnt);
    for (int t = 0; t < iters; ++t) {
        const float sc = buf_s[t * 33];
        const int ix = buf_i[t * 33];
        topk_insert_tail<KMAX>(ts, ti, (t < cnt && sc > ts[KMAX - 1]) ? sc : -INFINITY, ix);
    }
}

template <int D, int KMAX, typename QT>
MOBA_DEV void route_topk_fp32_tile(const QT* __restrict__ Q, const float* __restrict__ cent, int64_t N,
                                   int B, int top_k, int kv_group, int32_t* __restrict__ topk, int64_t h, int tile) {
    extern __shared__ __align__(16) float route_smem[];
    float (*q_s)[kRouteQ] = reinterpret_cast<float (*)[kRouteQ]>(route_smem);
    float (*c_s)[kRouteC] = reinterpret_cast<float (*)[kRouteC]>(route_smem + D * kRouteQ);
    float (*s_s)[kRouteC + 1] = reinterpret_cast<float (*)[kRouteC + 1]>(route_smem + D * (kRouteQ + kRouteC));
    float* sel_s = route_smem + D * (kRouteQ + kRouteC) + kRouteQ * (kRouteC + 1);   // [4 warps][33][33]
    int* sel_i = reinterpret_cast<int*>(sel_s + 4 * 33 * 33);

    const int tid = threadIdx.x;
    const int64_t r0 = (int64_t)tile * kRouteQ;
    const int n_blocks = (int)((N + B - 1) / B);
    const int width = top_k + 1;
    const QT* Qh = Q + h * N * D;
    __syncthreads();   // a persistent CTA's previous tile is done with the shared buffers
    const float* Ch = cent + (int64_t)(h / kv_group) * n_blocks * D;   // GQA: the query head's K/V head

    // stage the query tile transposed (fp32, exact)
    for (int e = tid; e < kRouteQ * (D / 8); e += kRouteThreads) {
        int r = e / (D / 8), cg = e % (D / 8);
        int64_t i = r0 + r;
        float x[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (i < N) ld8f(Qh + i * D + cg * 8, x);
#pragma unroll
        for (int c = 0; c < 8; ++c) q_s[cg * 8 + c][r] = x[c];
    }

    const int64_t my_i = r0 + tid;
    const int my_own = (int)(min64(my_i, N - 1) / B);
    const int64_t last_i = min64(r0 + kRouteQ, N) - 1;
    const int max_own = (int)(last_i / B);

    float ts[KMAX];
    int ti[KMAX];
#pragma unroll
    for (int u = 0; u < KMAX; ++u) {
        ts[u] = -INFINITY;
        ti[u] = 0x7fffffff;
    }

    // micro-tile: 4 queries x 8 centroids per thread
    const int qg = tid % 32;    // query group -> rows qg*4 .. +3
    const int cgp = tid / 32;   // centroid group -> cols cgp*8 .. +7 (warp-uniform)

    for (int c0 = 0; c0 < max_own; c0 += kRouteC) {
        __syncthreads();  // previous chunk's c_s / s_s readers are done
        for (int e = tid; e < kRouteC * D; e += kRouteThreads) {
            int c = e / D, dd = e % D;
            int j = c0 + c;
            c_s[dd][c] = (j < n_blocks) ? Ch[(int64_t)j * D + dd] : 0.f;
        }
        __syncthreads();
        float acc[4][8];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 8; ++b) acc[a][b] = 0.f;
#pragma unroll 8
        for (int dd = 0; dd < D; ++dd) {
            float4 qv = *reinterpret_cast<const float4*>(&q_s[dd][qg * 4]);
            float4 c0v = *reinterpret_cast<const float4*>(&c_s[dd][cgp * 8]);
            float4 c1v = *reinterpret_cast<const float4*>(&c_s[dd][cgp * 8 + 4]);
            float qa[4] = {qv.x, qv.y, qv.z, qv.w};
            float cb[8] = {c0v.x, c0v.y, c0v.z, c0v.w, c1v.x, c1v.y, c1v.z, c1v.w};
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 8; ++b) acc[a][b] = fmaf(qa[a], cb[b], acc[a][b]);
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 8; ++b) s_s[qg * 4 + a][cgp * 8 + b] = acc[a][b];
        __syncthreads();
        // selection: thread tid owns query r0 + tid; only strictly-past
        // blocks j < own compete (src/router.py:92)
        const int lim = (my_i < N) ? min(kRouteC, my_own - c0) : 0;
        {
            float sv[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) sv[c] = s_s[tid][c];
            select_chunk32<KMAX>(sv, c0, lim, ts, ti, sel_s + (tid & 31) + (tid >> 5) * 33 * 33,
                                 sel_i + (tid & 31) + (tid >> 5) * 33 * 33);
        }
    }

    if (my_i >= N) return;
    // keep the first top_k entries, sort indices ascending, append own block
#pragma unroll
    for (int u = 0; u < KMAX; ++u)
        if (u >= top_k) ti[u] = 0x7fffffff;
#pragma unroll
    for (int p = 0; p < KMAX; ++p) {
#pragma unroll
        for (int u = (p & 1); u + 1 < KMAX; u += 2) {
            int a = ti[u], b = ti[u + 1];
            ti[u] = min(a, b);
            ti[u + 1] = max(a, b);
        }
    }
    int32_t* row = topk + (h * N + my_i) * width;
    int nvalid = 0;
#pragma unroll
    for (int u = 0; u < KMAX; ++u) {
        if (ti[u] != 0x7fffffff) {
            row[u] = ti[u];
            ++nvalid;
        }
    }
    row[nvalid] = my_own;
    for (int s = nvalid + 1; s < width; ++s) row[s] = -1;
}


// tiles == nullptr: one CTA per (128-query tile, head) of the grid.
// tiles != nullptr: persistent CTAs walk the device list tiles[1 .. tiles[0]]
// of (head * n_tiles + tile) ids — the tiles the tensor-core router could
// not decide exactly (route_tc.cu), routed again here from scratch.
template <int D, int KMAX, typename QT>
__global__ void __launch_bounds__(kRouteThreads)
route_topk_fp32_kernel(const QT* __restrict__ Q, const float* __restrict__ cent, int64_t N,
                       int B, int top_k, int kv_group, int32_t* __restrict__ topk, const int* __restrict__ tiles,
                       const int* __restrict__ rows_count) {
    // tile-list mode runs only when the undecided rows are many per listed
    // tile (route_recheck_kernel takes them one by one otherwise)
    const int n_list = tiles == nullptr ? 1 : (rows_count != nullptr && *rows_count <= 16 * *tiles) ? 0 : *tiles;
    const int n_tiles = (int)((N + kRouteQ - 1) / kRouteQ);
    for (int li = tiles != nullptr ? (int)blockIdx.x : 0; li < n_list; li += (tiles != nullptr ? (int)gridDim.x : 1)) {
    const int tile_id = tiles != nullptr ? tiles[1 + li] : 0;
    route_topk_fp32_tile<D, KMAX, QT>(Q, cent, N, B, top_k, kv_group, topk,
                                      tiles != nullptr ? tile_id / n_tiles : (int64_t)blockIdx.y,
                                      tiles != nullptr ? tile_id % n_tiles : (int)blockIdx.x);
    }
}


// tensor-core routing (with the exactness guard): route_tc.cu

// ---------------------------------------------------------------- varlen
// build_varlen as a stable counting sort over query chunks:
//  count   : per (head, chunk of TQ queries) a shared-memory histogram over
//            blocks -> cc[h][chunk][b]
//  scan    : per (head, block) exclusive scan over chunks (in place) and
//            counts[b]; then offsets = exclusive scan over blocks
//  scatter : per (head, chunk) warps walk their runs of the chunk's
//            queries in ascending order, lanes = row slots; a row never repeats a block, so the
//            per-block cursors in shared memory are conflict free and each
//            block's slice comes out strictly ascending (src/router.py:145-148).

__global__ void varlen_count_kernel(const int32_t* __restrict__ topk, int64_t N, int width, int n_blocks,
                                    int TQ, int n_chunks, int32_t* __restrict__ cc, int* __restrict__ err) {
    extern __shared__ int hist[];
    const int64_t h = blockIdx.y;
    const int chunk = blockIdx.x;
    for (int b = threadIdx.x; b < n_blocks; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    const int64_t i0 = (int64_t)chunk * TQ;
    const int64_t i1 = min64(i0 + TQ, N);
    const int32_t* base = topk + h * N * width;
    // 8 loads in flight per thread before the shared-memory atomics
    const int64_t e_end = i1 * width;
    for (int64_t e0 = i0 * width + threadIdx.x; e0 < e_end; e0 += 8 * (int64_t)blockDim.x) {
        int v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t e = e0 + (int64_t)u * blockDim.x;
            v[u] = (e < e_end) ? __ldg(base + e) : -1;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int b = v[u];
            if (b >= n_blocks || b < -1) {
                atomicOr(err, 1);
            } else if (b >= 0) {
                atomicAdd(&hist[b], 1);
            }
        }
    }
    __syncthreads();
    int32_t* out = cc + (h * n_chunks + chunk) * (int64_t)n_blocks;
    for (int b = threadIdx.x; b < n_blocks; b += blockDim.x) out[b] = hist[b];
}

// Column scan split 4 ways: a CTA takes 32 block columns, its 4 warps each
// a quarter of the chunks (first pass: segment sums; second pass: rescan the
// segment from its base, the reads hit L2). The one-CTA-per-head scan had
// each thread walk all chunks of a column in dependent batches of 16 loads.
__global__ void __launch_bounds__(128)
varlen_scan_cols_kernel(int32_t* __restrict__ cc, int n_blocks, int n_chunks, int32_t* __restrict__ counts) {
    __shared__ int32_t part[4][32];
    const int64_t h = blockIdx.y;
    const int lane = threadIdx.x & 31, seg = threadIdx.x >> 5;
    const int b = blockIdx.x * 32 + lane;
    const int L = (n_chunks + 3) / 4;
    const int c_lo = min(n_chunks, seg * L), c_hi = min(n_chunks, (seg + 1) * L);
    int32_t* col = cc + h * (int64_t)n_chunks * n_blocks + b;
    int32_t sum = 0;
    if (b < n_blocks) {
        int c = c_lo;
        for (; c + 16 <= c_hi; c += 16) {
            int32_t v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) v[u] = col[(int64_t)(c + u) * n_blocks];
#pragma unroll
            for (int u = 0; u < 16; ++u) sum += v[u];
        }
        for (; c < c_hi; ++c) sum += col[(int64_t)c * n_blocks];
    }
    part[seg][lane] = sum;
    __syncthreads();
    if (b >= n_blocks) return;
    int32_t run = 0;
    for (int s2 = 0; s2 < seg; ++s2) run += part[s2][lane];
    if (seg == 3) counts[h * n_blocks + b] = run + sum;
    int c = c_lo;
    for (; c + 16 <= c_hi; c += 16) {
        int32_t v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = col[(int64_t)(c + u) * n_blocks];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            col[(int64_t)(c + u) * n_blocks] = run;
            run += v[u];
        }
    }
    for (; c < c_hi; ++c) {
        const int32_t v = col[(int64_t)c * n_blocks];
        col[(int64_t)c * n_blocks] = run;
        run += v;
    }
}

// per head: offsets = exclusive scan of the block counts, 1024 at a time
__global__ void __launch_bounds__(1024)
varlen_offsets_kernel(const int32_t* __restrict__ counts, int n_blocks, int32_t* __restrict__ offsets) {
    __shared__ int32_t warp_tot[32];
    __shared__ int32_t carry;
    const int64_t h = blockIdx.x;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int b0 = 0; b0 < n_blocks; b0 += 1024) {
        int b = b0 + threadIdx.x;
        int32_t v = (b < n_blocks) ? counts[h * n_blocks + b] : 0;
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
            warp_tot[lane] = t;  // inclusive
        }
        __syncthreads();
        int32_t excl = carry + (wid ? warp_tot[wid - 1] : 0) + x - v;
        if (b < n_blocks) offsets[h * n_blocks + b] = excl;
        __syncthreads();
        if (threadIdx.x == 0) carry += warp_tot[31];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(1024)
varlen_scan_kernel(int32_t* __restrict__ cc, int n_blocks, int n_chunks, int32_t* __restrict__ counts,
                   int32_t* __restrict__ offsets) {
    __shared__ int32_t warp_tot[32];
    __shared__ int32_t carry;
    const int64_t h = blockIdx.x;
    int32_t* cch = cc + h * (int64_t)n_chunks * n_blocks;
    // per block: exclusive scan over chunks, 16 chunk loads in flight
    for (int b = threadIdx.x; b < n_blocks; b += blockDim.x) {
        int32_t run = 0;
        int c = 0;
        for (; c + 16 <= n_chunks; c += 16) {
            int32_t v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) v[u] = cch[(int64_t)(c + u) * n_blocks + b];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                cch[(int64_t)(c + u) * n_blocks + b] = run;
                run += v[u];
            }
        }
        for (; c < n_chunks; ++c) {
            int32_t v = cch[(int64_t)c * n_blocks + b];
            cch[(int64_t)c * n_blocks + b] = run;
            run += v;
        }
        counts[h * n_blocks + b] = run;
    }
    __syncthreads();
    // offsets: exclusive scan of counts over blocks, 1024 at a time
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int b0 = 0; b0 < n_blocks; b0 += 1024) {
        int b = b0 + threadIdx.x;
        int32_t v = (b < n_blocks) ? counts[h * n_blocks + b] : 0;
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
            warp_tot[lane] = t;  // inclusive
        }
        __syncthreads();
        int32_t excl = carry + (wid ? warp_tot[wid - 1] : 0) + x - v;
        if (b < n_blocks) offsets[h * n_blocks + b] = excl;
        __syncthreads();
        if (threadIdx.x == 0) carry += warp_tot[31];
        __syncthreads();
    }
}

// The chunk's rows (TQ x width int32) are first staged in shared memory with
// coalesced loads that are all in flight together; the ordered walk then
// runs from shared memory.
__global__ void __launch_bounds__(128)
varlen_scatter_kernel(const int32_t* __restrict__ topk, int64_t N, int width, int n_blocks, int TQ,
                      int n_chunks, const int32_t* __restrict__ cc, const int32_t* __restrict__ offsets,
                      int32_t* __restrict__ flat, int32_t* __restrict__ row_pos) {
    extern __shared__ int32_t vsm[];
    int32_t* cursor = vsm;                   // [n_blocks]
    int32_t* rows_s = vsm + n_blocks;        // [TQ * width]
    const int64_t h = blockIdx.y;
    const int chunk = blockIdx.x;
    const int tid = threadIdx.x;
    const int32_t* ccc = cc + (h * n_chunks + chunk) * (int64_t)n_blocks;
    const int64_t i0 = (int64_t)chunk * TQ;
    const int64_t i1 = min64(i0 + TQ, N);
    const int nq = (int)(i1 - i0);
    for (int b = tid; b < n_blocks; b += blockDim.x) cursor[b] = offsets[h * n_blocks + b] + ccc[b];
    const int32_t* tk = topk + (h * N + i0) * width;
    for (int e = tid; e < nq * width; e += blockDim.x) rows_s[e] = __ldg(tk + e);
    __syncthreads();
    int32_t* rp = row_pos + (h * N + i0) * width;
    int32_t* fl = flat + h * N * width;
    if (tid < 32) {
        // Entries in (query, slot) order, 32 per step: lanes holding the same
        // block (__match_any_sync) rank themselves by lane = entry order =
        // query order (a row never repeats a block), so every block's slice
        // comes out strictly ascending, as the reference's cursor walk
        // (src/router.py:143-148).
        const int lane = tid;
        const int ne = nq * width;
        const unsigned lt = (1u << lane) - 1u;
        for (int e0 = 0; e0 < ne; e0 += 32) {
            const int e = e0 + lane;
            const int32_t b = (e < ne) ? rows_s[e] : -1;
            const unsigned grp = __match_any_sync(0xffffffffu, b);
            int32_t p = -1;
            if (b >= 0) {
                const int32_t base = cursor[b];
                p = base + __popc(grp & lt);
                fl[p] = (int32_t)(i0 + e / width);
            }
            __syncwarp();
            if (b >= 0 && (grp & lt) == 0) cursor[b] += __popc(grp);   // group leader advances the cursor
            if (e < ne) rows_s[e] = p;
            __syncwarp();
        }
    }
    __syncthreads();
    for (int e = tid; e < nq * width; e += blockDim.x) rp[e] = rows_s[e];
}

// Wide-chunk scatter: chunks of up to 2048 queries walked by W warps at once
// (a warp per contiguous run of the chunk's rows). The per-warp cursors are
// 16-bit offsets relative to the chunk's 32-bit base per block, two warps
// per shared word (warp 2i in the low half, 2i+1 in the high half; a chunk
// holds <= 16384 queries, so no half carries into the other), so the
// chunk setup is (1 + W/2) words per block instead of W, amortised over
// 4-16x more entries than a 128-query chunk; each warp then walks its rows
// in ascending order (src/router.py:143-148).
template <int W>
__global__ void __launch_bounds__(32 * W)
varlen_scatter_w_kernel(const int32_t* __restrict__ topk, int64_t N, int width, int n_blocks, int TQ,
                        int n_chunks, const int32_t* __restrict__ cc, const int32_t* __restrict__ offsets,
                        int32_t* __restrict__ flat, int32_t* __restrict__ row_pos) {
    constexpr int NT = 32 * W, P = W / 2;
    extern __shared__ int32_t vsm[];
    __shared__ int n_hi_s;                                            // 1 + the chunk's largest block
    const int n4 = (n_blocks + 3) & ~3;
    uint32_t* rel = reinterpret_cast<uint32_t*>(vsm);                 // [P][n4]
    int32_t* base = vsm + P * n4;                                     // [n_blocks]
    int32_t* rows_s = base + n4;                                      // [TQ * width]
    const int64_t h = blockIdx.y;
    const int chunk = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t i0 = (int64_t)chunk * TQ;
    const int nq = (int)(min64(i0 + TQ, N) - i0);
    const int ne = nq * width;
    const int32_t* tk = topk + (h * N + i0) * width;
    {
        int e = tid;
        for (; e + 7 * NT < ne; e += 8 * NT) {
            int v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(tk + e + u * NT);
#pragma unroll
            for (int u = 0; u < 8; ++u) rows_s[e + u * NT] = v[u];
        }
        for (; e < ne; e += NT) rows_s[e] = __ldg(tk + e);
    }
    for (int b = tid; b < P * n4 / 4; b += NT) reinterpret_cast<uint4*>(rel)[b] = make_uint4(0u, 0u, 0u, 0u);
    if (tid == 0) n_hi_s = 0;
    __syncthreads();
    const int qw = (nq + W - 1) / W;
    const int e_lo = min(nq, warp * qw) * width, e_hi = min(nq, (warp + 1) * qw) * width;
    uint32_t* my = rel + (warp >> 1) * n4;
    const int sh = (warp & 1) * 16;
    int bmax = -1;
    for (int e = e_lo + lane; e < e_hi; e += 32) {
        const int32_t b = rows_s[e];
        if (b >= 0) atomicAdd(&my[b], 1u << sh);
        bmax = max(bmax, b);
    }
    bmax = __reduce_max_sync(0xffffffffu, bmax);
    if (lane == 0) atomicMax(&n_hi_s, bmax + 1);
    __syncthreads();
    // per block the chunk touches (causal plans: blocks <= the chunk's last
    // query block): the chunk's base, then each warp's exclusive offset
    const int n_hi = n_hi_s;
    const int32_t* ccc = cc + (h * n_chunks + chunk) * (int64_t)n_blocks;
    const int32_t* offh = offsets + h * n_blocks;
    for (int b0 = tid; b0 < n_hi; b0 += 4 * NT) {
        int32_t r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int b = b0 + u * NT;
            r[u] = b < n_hi ? __ldg(offh + b) + __ldg(ccc + b) : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int b = b0 + u * NT;
            if (b < n_hi) {
                base[b] = r[u];
                uint32_t w[P];
#pragma unroll
                for (int p = 0; p < P; ++p) w[p] = rel[p * n4 + b];
                uint32_t run = 0;
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const uint32_t lo = w[p] & 0xffffu;
                    rel[p * n4 + b] = run | ((run + lo) << 16);
                    run += lo + (w[p] >> 16);
                }
            }
        }
    }
    __syncthreads();
    // the walk: one row per step, lane = slot. A row never repeats a block,
    // so the lanes of a step hit distinct cursors (no match / rank step);
    // consecutive steps are ordered by the warp's in-order shared atomics
    int32_t* fl = flat + h * N * width;
    const int r_lo = e_lo / width, r_hi = e_hi / width;
#pragma unroll 4
    for (int r = r_lo; r < r_hi; ++r) {
        if (lane < width) {
            const int e = r * width + lane;
            const int32_t b = rows_s[e];
            int32_t p = -1;
            if (b >= 0) {
                const uint32_t old = atomicAdd(&my[b], 1u << sh);
                p = base[b] + (int32_t)((old >> sh) & 0xffffu);
                fl[p] = (int32_t)(i0 + r);
            }
            rows_s[e] = p;
        }
    }
    __syncthreads();
    int32_t* rp = row_pos + (h * N + i0) * width;
    for (int e = tid; e < ne; e += NT) rp[e] = rows_s[e];
}

// row_pos from an arbitrary (validated) plan: binary search of query i in
// block b's ascending slice.
__global__ void plan_row_pos_kernel(const int32_t* __restrict__ topk, const int32_t* __restrict__ counts,
                                    const int32_t* __restrict__ offsets, const int32_t* __restrict__ flat,
                                    int64_t N, int width, int n_blocks, int32_t* __restrict__ row_pos) {
    const int64_t h = blockIdx.y;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= N * width) return;
    const int64_t i = e / width;
    int32_t b = topk[h * N * width + e];
    int32_t p = -1;
    if (b >= 0) {
        const int32_t* sl = flat + h * N * width + offsets[h * n_blocks + b];
        int lo = 0, hi = counts[h * n_blocks + b];
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (sl[mid] < i) lo = mid + 1; else hi = mid;
        }
        if (lo < counts[h * n_blocks + b] && sl[lo] == i) p = offsets[h * n_blocks + b] + lo;
    }
    row_pos[h * N * width + e] = p;
}

// ---------------------------------------------------------------- validation
// flags: bit0 range, bit1 causality, bit2 duplicate, bit3 prefix/total,
// bit4 slice order / range, bit5 (query, block) of topk absent from flat
__global__ void validate_rows_kernel(const int32_t* __restrict__ topk, int64_t N, int width, int B,
                                     int n_blocks, unsigned long long* __restrict__ valid_count,
                                     int* __restrict__ flags) {
    const int64_t h = blockIdx.y;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int32_t* row = topk + (h * N + i) * width;
    int nv = 0, f = 0;
    const int own = (int)(i / B);
    for (int s = 0; s < width; ++s) {
        int b = row[s];
        if (b < -1 || b >= n_blocks) f |= 1;
        if (b >= 0) {
            ++nv;
            if (b > own) f |= 2;
            for (int t = 0; t < s; ++t)
                if (row[t] == b) f |= 4;
        }
    }
    if (f) atomicOr(flags, f);
    atomicAdd(&valid_count[h], (unsigned long long)nv);
}

__global__ void validate_blocks_kernel(const int32_t* __restrict__ counts, const int32_t* __restrict__ offsets,
                                       int n_blocks, const unsigned long long* __restrict__ valid_count,
                                       int* __restrict__ flags) {
    const int64_t h = blockIdx.x;
    if (threadIdx.x != 0) return;
    long long run = 0;
    int f = 0;
    for (int b = 0; b < n_blocks; ++b) {
        int32_t c = counts[h * n_blocks + b];
        if (c < 0) f |= 8;
        if (offsets[h * n_blocks + b] != run) f |= 8;
        run += c;
    }
    if ((unsigned long long)run != valid_count[h]) f |= 8;
    if (f) atomicOr(flags, f);
}

__global__ void validate_flat_kernel(const int32_t* __restrict__ counts, const int32_t* __restrict__ offsets,
                                     const int32_t* __restrict__ flat, int64_t N, int width, int B,
                                     int n_blocks, int* __restrict__ flags) {
    const int64_t h = blockIdx.y;
    const int b = blockIdx.x;
    const int32_t c = counts[h * n_blocks + b];
    const int32_t o = offsets[h * n_blocks + b];
    if (c < 0 || o < 0 || (int64_t)o + c > N * width) return;  // reported by the blocks check
    const int32_t* sl = flat + h * N * width + o;
    int f = 0;
    for (int p = threadIdx.x; p < c; p += blockDim.x) {
        int32_t q = sl[p];
        if (q < (int64_t)b * B || q >= N) f |= 16;
        if (p > 0 && sl[p - 1] >= q) f |= 16;
    }
    if (f) atomicOr(flags, f);
}

// bit5: every valid (query, block) entry of topk must appear in block's
// slice. With the totals equal (bit3) and slices strictly ascending (bit4)
// this makes the two layouts describe the same (query, block) set.
__global__ void validate_membership_kernel(const int32_t* __restrict__ topk, const int32_t* __restrict__ counts,
                                           const int32_t* __restrict__ offsets, const int32_t* __restrict__ flat,
                                           int64_t N, int width, int n_blocks, int* __restrict__ flags) {
    const int64_t h = blockIdx.y;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= N * width) return;
    const int32_t b = topk[h * N * width + e];
    if (b < 0) return;
    const int32_t i = (int32_t)(e / width);
    const int32_t* sl = flat + h * N * width + offsets[h * n_blocks + b];
    const int c = counts[h * n_blocks + b];
    int lo = 0, hi = c;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (sl[mid] < i) lo = mid + 1; else hi = mid;
    }
    if (lo >= c || sl[lo] != i) atomicOr(flags, 32);
}

// varlen workspace layout: [err int | cc int32 (bh * n_chunks * n)]
struct VarlenGeom {
    int TQ;
    int n_chunks;
    int n_blocks;
    int W;   // walking warps of the wide-chunk scatter (0: the one-warp capacity fallback)
};

constexpr size_t kVarlenSmem = 227 * 1024 - 64;   // + the kernel's static word

// chunk size the wide scatter grows towards: n/2 queries, clamped to
// [512, 2048] (measured, b2 x h16 d64 B128 k8: 64K 512 -> 0.174 ms, 256K
// 1024 -> 0.65 ms, 512K 2048 -> 1.58 ms; smaller chunks repeat the O(n)
// cursor setup more often, larger ones leave too few CTAs per SM)
static int64_t varlen_tq_target(int n_blocks) {
    return std::min<int64_t>(2048, std::max<int64_t>(512, n_blocks / 2));
}

static size_t varlen_wide_smem(int64_t tq, int w, int n_blocks, int width) {
    return ((size_t)(1 + w / 2) * ((n_blocks + 3) & ~3) + (size_t)tq * width) * sizeof(int32_t);
}

// The chunk geometry of one varlen call (the workspace query uses the same
// function, so the chunk-count matrix it sizes is exact): chunks of >= 128
// queries with at most 4M chunk-count entries per head; then, for the wide
// scatter, the most walking warps whose cursor words fit in shared memory
// and chunks grown towards varlen_tq_target while the grid keeps >= 2 CTAs
// per SM.
static VarlenGeom varlen_geom(int64_t bh, int64_t n_tokens, int block_size, int width) {
    VarlenGeom g;
    g.n_blocks = (int)ceil_div(n_tokens, block_size);
    int64_t tq = 128;
    while (ceil_div(n_tokens, tq) * (int64_t)g.n_blocks > (4ll << 20) && tq < (1 << 20)) tq *= 2;
    int W = 16;
    while (W > 2 && varlen_wide_smem(tq, W, g.n_blocks, width) > kVarlenSmem) W /= 2;
    if (tq > 16384 || varlen_wide_smem(tq, W, g.n_blocks, width) > kVarlenSmem) W = 0;
    if (W > 0) {
        const int64_t target = varlen_tq_target(g.n_blocks);
        while (tq < target && bh * ceil_div(n_tokens, 2 * tq) >= 2 * kNumSMs &&
               varlen_wide_smem(2 * tq, W, g.n_blocks, width) <= kVarlenSmem)
            tq *= 2;
    }
    g.W = W;
    g.TQ = (int)tq;
    g.n_chunks = (int)ceil_div(n_tokens, tq);
    return g;
}

static int run_varlen(const int32_t* topk, int64_t bh, int64_t N, int width, int B, int32_t* counts,
                      int32_t* offsets, int32_t* flat, int32_t* row_pos, void* ws, size_t ws_bytes,
                      cudaStream_t s, bool sync_range_check) {
    const VarlenGeom g = varlen_geom(bh, N, B, width);
    if (g.n_blocks > 16384) return MOBA_ERR_UNSUPPORTED;
    size_t need = 256 + (size_t)bh * g.n_chunks * g.n_blocks * sizeof(int32_t);
    if (ws_bytes < need) return MOBA_ERR_WORKSPACE;
    int* err = (int*)ws;
    int32_t* cc = (int32_t*)((char*)ws + 256);
    const int W = g.W;
    StageTimer tm(T_VARLEN, s);
    cudaMemsetAsync(err, 0, sizeof(int), s);
    size_t hsmem = (size_t)g.n_blocks * sizeof(int);
    if (hsmem > 48 * 1024)
        cudaFuncSetAttribute(varlen_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsmem);
    varlen_count_kernel<<<dim3(g.n_chunks, (unsigned)bh), 128, hsmem, s>>>(topk, N, width, g.n_blocks, g.TQ,
                                                                        g.n_chunks, cc, err);
    int st = check_launch("varlen_count_kernel");
    if (st) return st;
    if (sync_range_check) {
        int herr = 0;
        cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        if (herr) return MOBA_ERR_PLAN;
    }
    if (g.n_chunks >= 64) {
        varlen_scan_cols_kernel<<<dim3((unsigned)ceil_div(g.n_blocks, 32), (unsigned)bh), 128, 0, s>>>(
            cc, g.n_blocks, g.n_chunks, counts);
        varlen_offsets_kernel<<<(unsigned)bh, 1024, 0, s>>>(counts, g.n_blocks, offsets);
        st = check_launch("varlen_scan_cols_kernel", 2);
    } else {
        varlen_scan_kernel<<<(unsigned)bh, 1024, 0, s>>>(cc, g.n_blocks, g.n_chunks, counts, offsets);
        st = check_launch("varlen_scan_kernel");
    }
    if (st) return st;
    if (W > 0) {
        const size_t wsmem = varlen_wide_smem(g.TQ, W, g.n_blocks, width);
        switch (W) {
#define MOBA_SCATTER_W(w)                                                                                       \
    case w:                                                                                                     \
        cudaFuncSetAttribute(varlen_scatter_w_kernel<w>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsmem); \
        varlen_scatter_w_kernel<w><<<dim3(g.n_chunks, (unsigned)bh), 32 * w, wsmem, s>>>(                      \
            topk, N, width, g.n_blocks, g.TQ, g.n_chunks, cc, offsets, flat, row_pos);                          \
        break;
            MOBA_SCATTER_W(16)
            MOBA_SCATTER_W(8)
            MOBA_SCATTER_W(4)
            MOBA_SCATTER_W(2)
#undef MOBA_SCATTER_W
        }
        return check_launch("varlen_scatter_w_kernel");
    }
    // capacity fallback (the per-warp cursor words do not fit): one walking warp
    const size_t ssmem = hsmem + (size_t)g.TQ * width * sizeof(int32_t);
    if (ssmem > 48 * 1024) {
        if (ssmem > 227 * 1024) return MOBA_ERR_UNSUPPORTED;
        cudaFuncSetAttribute(varlen_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssmem);
    }
    varlen_scatter_kernel<<<dim3(g.n_chunks, (unsigned)bh), 128, ssmem, s>>>(
        topk, N, width, g.n_blocks, g.TQ, g.n_chunks, cc, offsets, flat, row_pos);
    return check_launch("varlen_scatter_kernel");
}

size_t route_tc_ws_bytes(int64_t bh, int64_t N, int B);
template <int D, int KMAX>
int launch_route_tc(const void* q, const float* cent, int64_t bh, int kv_group, int64_t N, int B, int top_k,
                    int32_t* topk, void* ws, cudaStream_t s);

// exact fp32 re-routing of the tiles listed in `tiles` (count, then ids)
template <int D, int KMAX>
int launch_route_fp32_tiles(const void* q, const float* cent, int64_t bh, int kv_group, int64_t N, int B, int top_k,
                            int32_t* topk, const int* tiles, const int* rows_count, cudaStream_t s) {
    const size_t fsmem = (size_t)(D * (kRouteQ + kRouteC) + kRouteQ * (kRouteC + 1) + 2 * 4 * 33 * 33) * sizeof(float);
    auto kern = route_topk_fp32_kernel<D, KMAX, __nv_bfloat16>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem);
    const int64_t n_tiles = bh * ceil_div(N, kRouteQ);
    const unsigned grid = (unsigned)std::min<int64_t>(n_tiles, 2 * kNumSMs);
    kern<<<grid, kRouteThreads, fsmem, s>>>((const __nv_bfloat16*)q, cent, N, B, top_k, kv_group, topk, tiles,
                                            rows_count);
    return check_launch("route_topk_fp32_kernel (tile list)");
}
#define MOBA_RF_INST(D, K)                                                                                       \
    template int launch_route_fp32_tiles<D, K>(const void*, const float*, int64_t, int, int64_t, int, int,      \
                                               int32_t*, const int*, const int*, cudaStream_t);
MOBA_RF_INST(64, 1) MOBA_RF_INST(64, 2) MOBA_RF_INST(64, 4) MOBA_RF_INST(64, 8) MOBA_RF_INST(64, 16) MOBA_RF_INST(64, 32)
MOBA_RF_INST(128, 1) MOBA_RF_INST(128, 2) MOBA_RF_INST(128, 4) MOBA_RF_INST(128, 8) MOBA_RF_INST(128, 16)
MOBA_RF_INST(128, 32)
#undef MOBA_RF_INST

template <int D, int KMAX>
static int launch_route(const void* q, bool q_f32, const float* cent, int64_t bh, int64_t N, int B, int top_k,
                        int mode, int kv_group, int32_t* topk, void* split_ws, cudaStream_t s) {
    dim3 grid((unsigned)ceil_div(N, kRouteQ), (unsigned)bh);
    const size_t fsmem = (size_t)(D * (kRouteQ + kRouteC) + kRouteQ * (kRouteC + 1) + 2 * 4 * 33 * 33) * sizeof(float);
    if (q_f32) {
        // fp32 queries (numpy f32 / f64 callers): exact fp32 products, no bf16 rounding before routing
        if (mode != MOBA_ROUTE_FP32) return MOBA_ERR_CONFIG;
        auto kern = route_topk_fp32_kernel<D, KMAX, float>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem);
        kern<<<grid, kRouteThreads, fsmem, s>>>((const float*)q, cent, N, B, top_k, kv_group, topk, nullptr, nullptr);
        return check_launch("route_topk_fp32_kernel");
    }
    if (mode == MOBA_ROUTE_TC) return launch_route_tc<D, KMAX>(q, cent, bh, kv_group, N, B, top_k, topk, split_ws, s);
    auto kern = route_topk_fp32_kernel<D, KMAX, __nv_bfloat16>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem);
    kern<<<grid, kRouteThreads, fsmem, s>>>((const __nv_bfloat16*)q, cent, N, B, top_k, kv_group, topk, nullptr, nullptr);
    return check_launch("route_topk_fp32_kernel");
}

template <int D>
static int dispatch_route_k(const void* q, bool q_f32, const float* cent, int64_t bh, int64_t N, int B, int top_k,
                            int mode, int kv_group, int32_t* topk, void* split_ws, cudaStream_t s) {
#define MOBA_ROUTE_K(KM) launch_route<D, KM>(q, q_f32, cent, bh, N, B, top_k, mode, kv_group, topk, split_ws, s)
    if (top_k <= 1) return MOBA_ROUTE_K(1);
    if (top_k <= 2) return MOBA_ROUTE_K(2);
    if (top_k <= 4) return MOBA_ROUTE_K(4);
    if (top_k <= 8) return MOBA_ROUTE_K(8);
    if (top_k <= 16) return MOBA_ROUTE_K(16);
    if (top_k <= 32) return MOBA_ROUTE_K(32);
#undef MOBA_ROUTE_K
    return MOBA_ERR_UNSUPPORTED;
}

}  // namespace moba

using namespace moba;

// workspace: [varlen: err | chunk counts] [route tc: bf16 centroid split 3 x bh x n x 128]
static size_t varlen_ws_bytes(int64_t bh, int64_t n_tokens, int block_size, int width) {
    const VarlenGeom g = varlen_geom(bh, n_tokens, block_size, width);
    return align_up(256 + (size_t)bh * g.n_chunks * g.n_blocks * sizeof(int32_t), 1024);
}

extern "C" size_t moba_route_workspace_size(int64_t bh, int64_t n_tokens, int block_size, int top_k) {
    if (block_size < 1 || n_tokens < 1 || top_k < 0) return 0;
    return varlen_ws_bytes(bh, n_tokens, block_size, top_k + 1) + route_tc_ws_bytes(bh, n_tokens, block_size);
}

static int route_impl(const void* q, bool q_f32, const float* centroids, int64_t bh, int kv_group, int64_t n_tokens,
                      int head_dim, int block_size, int top_k, int mode, int32_t* topk, int32_t* counts,
                      int32_t* offsets, int32_t* flat, int32_t* row_pos, void* workspace, size_t workspace_bytes,
                      void* stream) {
    clear_last_error();
    if (bh < 1 || bh > 65535 || n_tokens < 1 || block_size < 1) return MOBA_ERR_SHAPE;
    if (kv_group < 1 || bh % kv_group != 0) return MOBA_ERR_SHAPE;
    if (top_k < 1) return MOBA_ERR_CONFIG;
    if (top_k > 31) return MOBA_ERR_UNSUPPORTED;
    if (mode != MOBA_ROUTE_FP32 && mode != MOBA_ROUTE_TC) return MOBA_ERR_CONFIG;
    cudaStream_t s = (cudaStream_t)stream;
    int st;
    {
    StageTimer tm(T_ROUTE, s);
    if (workspace_bytes < moba_route_workspace_size(bh, n_tokens, block_size, top_k)) return MOBA_ERR_WORKSPACE;
    void* split_ws = (char*)workspace + varlen_ws_bytes(bh, n_tokens, block_size, top_k + 1);
    if (head_dim == 64)
        st = dispatch_route_k<64>(q, q_f32, centroids, bh, n_tokens, block_size, top_k, mode, kv_group, topk,
                                  split_ws, s);
    else if (head_dim == 128)
        st = dispatch_route_k<128>(q, q_f32, centroids, bh, n_tokens, block_size, top_k, mode, kv_group, topk,
                                   split_ws, s);
    else return MOBA_ERR_UNSUPPORTED;
    }
    if (st) return st;
    return run_varlen(topk, bh, n_tokens, top_k + 1, block_size, counts, offsets, flat, row_pos, workspace,
                      workspace_bytes, s, false);
}

extern "C" int moba_route_gqa(const void* q, const float* centroids, int64_t bh, int kv_group, int64_t n_tokens,
                              int head_dim, int block_size, int top_k, int mode, int32_t* topk, int32_t* counts,
                              int32_t* offsets, int32_t* flat, int32_t* row_pos, void* workspace,
                              size_t workspace_bytes, void* stream) {
    return route_impl(q, false, centroids, bh, kv_group, n_tokens, head_dim, block_size, top_k, mode, topk, counts,
                      offsets, flat, row_pos, workspace, workspace_bytes, stream);
}

extern "C" int moba_route_f32(const float* q, const float* centroids, int64_t bh, int kv_group, int64_t n_tokens,
                              int head_dim, int block_size, int top_k, int32_t* topk, int32_t* counts,
                              int32_t* offsets, int32_t* flat, int32_t* row_pos, void* workspace,
                              size_t workspace_bytes, void* stream) {
    return route_impl(q, true, centroids, bh, kv_group, n_tokens, head_dim, block_size, top_k, MOBA_ROUTE_FP32, topk,
                      counts, offsets, flat, row_pos, workspace, workspace_bytes, stream);
}

extern "C" int moba_route(const void* q, const float* centroids, int64_t bh, int64_t n_tokens, int head_dim,
                          int block_size, int top_k, int mode, int32_t* topk, int32_t* counts,
                          int32_t* offsets, int32_t* flat, int32_t* row_pos, void* workspace,
                          size_t workspace_bytes, void* stream) {
    return moba_route_gqa(q, centroids, bh, 1, n_tokens, head_dim, block_size, top_k, mode, topk, counts, offsets,
                          flat, row_pos, workspace, workspace_bytes, stream);
}

extern "C" int moba_varlen(const int32_t* topk, int64_t bh, int64_t n_tokens, int width, int block_size,
                           int32_t* counts, int32_t* offsets, int32_t* flat, int32_t* row_pos, void* workspace,
                           size_t workspace_bytes, void* stream) {
    clear_last_error();
    if (bh < 1 || bh > 65535 || n_tokens < 1 || block_size < 1 || width < 1) return MOBA_ERR_SHAPE;
    if (width > 32) return MOBA_ERR_UNSUPPORTED;
    return run_varlen(topk, bh, n_tokens, width, block_size, counts, offsets, flat, row_pos, workspace,
                      workspace_bytes, (cudaStream_t)stream, true);
}

extern "C" int moba_plan_row_pos(const int32_t* topk, const int32_t* counts, const int32_t* offsets,
                                 const int32_t* flat, int64_t bh, int64_t n_tokens, int width, int block_size,
                                 int32_t* row_pos, void* stream) {
    clear_last_error();
    if (bh < 1 || bh > 65535 || n_tokens < 1 || block_size < 1 || width < 1) return MOBA_ERR_SHAPE;
    int n_blocks = (int)ceil_div(n_tokens, block_size);
    dim3 grid((unsigned)ceil_div(n_tokens * width, 256), (unsigned)bh);
    plan_row_pos_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(topk, counts, offsets, flat, n_tokens, width,
                                                                n_blocks, row_pos);
    return check_launch("plan_row_pos_kernel");
}

extern "C" int moba_validate_plan(const int32_t* topk, const int32_t* counts, const int32_t* offsets,
                                  const int32_t* flat, int64_t bh, int64_t n_tokens, int width, int block_size,
                                  void* workspace, size_t workspace_bytes, void* stream) {
    clear_last_error();
    if (bh < 1 || bh > 65535 || n_tokens < 1 || block_size < 1 || width < 1) return MOBA_ERR_SHAPE;
    size_t need = 256 + (size_t)bh * sizeof(unsigned long long);
    if (workspace_bytes < need) return MOBA_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    int n_blocks = (int)ceil_div(n_tokens, block_size);
    int* flags = (int*)workspace;
    unsigned long long* vc = (unsigned long long*)((char*)workspace + 256);
    cudaMemsetAsync(workspace, 0, need, s);
    validate_rows_kernel<<<dim3((unsigned)ceil_div(n_tokens, 256), (unsigned)bh), 256, 0, s>>>(
        topk, n_tokens, width, block_size, n_blocks, vc, flags);
    check_launch("validate_rows_kernel");
    validate_blocks_kernel<<<(unsigned)bh, 32, 0, s>>>(counts, offsets, n_blocks, vc, flags);
    int hf = 0;
    cudaMemcpyAsync(&hf, flags, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    int st = check_launch("validate_plan");
    if (st) return st;
    if (hf) return MOBA_ERR_PLAN;
    // slices are only inspected once counts/offsets are known consistent
    validate_flat_kernel<<<dim3((unsigned)n_blocks, (unsigned)bh), 256, 0, s>>>(counts, offsets, flat, n_tokens,
                                                                             width, block_size, n_blocks, flags);
    cudaMemcpyAsync(&hf, flags, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    st = check_launch("validate_flat_kernel");
    if (st) return st;
    if (hf) return MOBA_ERR_PLAN;
    // membership once the slices are known sorted and in range
    validate_membership_kernel<<<dim3((unsigned)ceil_div(n_tokens * width, 256), (unsigned)bh), 256, 0, s>>>(
        topk, counts, offsets, flat, n_tokens, width, n_blocks, flags);
    cudaMemcpyAsync(&hf, flags, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    st = check_launch("validate_membership_kernel");
    if (st) return st;
    if (hf) set_last_error("a (query, block) entry of topk_indices is missing from its block's flat_queries slice");
    return hf ? MOBA_ERR_PLAN : MOBA_OK;
}
