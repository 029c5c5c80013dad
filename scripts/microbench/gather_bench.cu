// Gather throughput per SM: 128 random 128-B rows (x2 tensors) per "tile" into
// SW128 smem, different mechanisms, 148 CTAs, back-to-back tiles.
#include "../../paper_2511_11571_b200/csrc/sm100.cuh"
#include <cuda.h>
#include <cstdio>
#include <vector>
using namespace moba;
using namespace moba::sm100;

// mode 0: cp.async, `nw` warps, coalesced (8 lanes / row); wait_group per tile
// mode 1: LDG.128 + STS.128 by `nw` warps
// mode 2: TMA gather4 issued by one warp, `depth` tiles in flight
__global__ void gather(const __nv_bfloat16* __restrict__ A, const __nv_bfloat16* __restrict__ Bt,
                       const int* __restrict__ rows, int nrows_total, int tiles, int mode, int nw,
                       const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                       long long* cyc, float* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar[4];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1); fence_mbar_init(); }
    __syncthreads();
    long long t0 = clock64();
    const int* rr = rows + (blockIdx.x * 997) % (nrows_total - tiles * 128);
    float acc = 0.f;
    if (mode == 0 || mode == 1) {
        if (warp < nw) {
            const int sub = lane % 8, rsub = lane / 8;
            for (int t = 0; t < tiles; ++t) {
                const uint32_t base = smem_u32(buf) + (t & 1) * 32768;
                for (int i = warp; i < 32; i += nw) {
                    const int r = 4 * i + rsub;
                    const int q = rr[t * 128 + r];
                    const uint32_t off = sw128_off(r, sub * 8, 128);
                    if (mode == 0) {
                        cp_async16(base + off, A + (int64_t)q * 64 + sub * 8);
                        cp_async16(base + 16384 + off, Bt + (int64_t)q * 64 + sub * 8);
                    } else {
                        uint4 va = *reinterpret_cast<const uint4*>(A + (int64_t)q * 64 + sub * 8);
                        uint4 vb = *reinterpret_cast<const uint4*>(Bt + (int64_t)q * 64 + sub * 8);
                        sts128(base + off, va);
                        sts128(base + 16384 + off, vb);
                    }
                }
                if (mode == 0) { cp_async_commit(); cp_async_wait<1>(); }
            }
            if (mode == 0) cp_async_wait<0>();
        }
    } else {
        const int depth = nw;  // tiles in flight
        if (warp == 0) {
            for (int t = 0; t < tiles; ++t) {
                const int s = t % depth;
                if (t >= depth) mbar_wait(&bar[s], ((t - depth) / depth) & 1);
                const uint32_t base = smem_u32(buf) + s * 32768;
                if (lane == 0) mbar_expect_tx(&bar[s], 32768);
                __syncwarp();
                const int* q = rr + t * 128 + 4 * lane;
                tma_gather4(base + 4 * lane * 128, &ma, 0, q[0], q[1], q[2], q[3], &bar[s]);
                tma_gather4(base + 16384 + 4 * lane * 128, &mb, 0, q[0], q[1], q[2], q[3], &bar[s]);
            }
            for (int t = tiles - depth; t < tiles; ++t) if (t >= 0) mbar_wait(&bar[t % depth], (t / depth) & 1);
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (acc == 1.f) sink[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
    const int R = 16 * 8192;  // 16 heads x 8K rows of 64 bf16 = 16 MB per tensor
    __nv_bfloat16 *a, *b; cudaMalloc(&a, (size_t)R * 128); cudaMalloc(&b, (size_t)R * 128);
    cudaMemset(a, 0, (size_t)R * 128); cudaMemset(b, 0, (size_t)R * 128);
    const int NT = 200 * 128 + 200000;
    std::vector<int> rows(NT);
    unsigned s = 12345;
    for (auto& x : rows) { s = s * 1664525u + 1013904223u; x = (s >> 8) % R; }
    int* dr; cudaMalloc(&dr, NT * 4); cudaMemcpy(dr, rows.data(), NT * 4, cudaMemcpyHostToDevice);
    long long* dc; cudaMalloc(&dc, 148 * 8); float* sink; cudaMalloc(&sink, 64);
    void* fn; cudaDriverEntryPointQueryResult q; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)fn;
    CUtensorMap ma, mb; cuuint64_t dims[2] = {64, (cuuint64_t)R}, st[1] = {128}; cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
    enc(&ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, b, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
    const int tiles = 200;
    struct { const char* n; int mode, nw; } cs[] = {{"cp.async 8 warps", 0, 8}, {"cp.async 16 warps", 0, 16}, {"cp.async 32 warps", 0, 32},
                                                    {"ldg+sts 32 warps", 1, 32}};
    for (auto& c : cs) {
        for (int rep = 0; rep < 2; ++rep) gather<<<148, 1024, 136 * 1024>>>(a, b, dr, NT, tiles, c.mode, c.nw, ma, mb, dc, sink);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<long long> h(148); cudaMemcpy(h.data(), dc, 148 * 8, cudaMemcpyDeviceToHost);
        long long mx = 0; for (auto x : h) mx = x > mx ? x : mx;
        printf("%-22s %s: %.0f cycles/tile (32 KB) -> %.1f B/clk/SM\n", c.n, cudaGetErrorString(e), (double)mx / tiles, 32768.0 * tiles / mx);
    }
    return 0;
}
