// Microbenchmark: steady-state gather throughput per SM with several 128-row
// (16 KB) batches in flight: TMA tile::gather4 issued by one lane vs
// cp.async (LDGSTS, 8 lanes per 128-B row) issued by W warps.
#include "../../paper_2511_11571_b200/csrc/sm100.cuh"
#include <cuda.h>
#include <cstdio>
#include <vector>
using namespace moba;
using namespace moba::sm100;
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__device__ void tma_g4(uint32_t dst, const CUtensorMap* map, int c0, int r0, int r1, int r2, int r3, uint64_t* bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                 :: "r"(dst), "l"(map), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar)) : "memory");
}
constexpr int S = 4;
__global__ void g4_kernel(const __grid_constant__ CUtensorMap map4, const int* rows, int nrows_total, int iters, long long* cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar[S];
    if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1); fence_mbar_init(); }
    __syncthreads();
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int it = 0; it < iters; ++it) {
            const int s = it % S;
            if (it >= S) mbar_wait(&bar[s], ((it / S) - 1) & 1);
            mbar_expect_tx(&bar[s], 128 * 128);
            const unsigned base = (blockIdx.x * 977u + it * 128u);
#define HROW(r) (int)(((base + (r)) * 2654435761u) % 131072u)
            for (int r = 0; r < 128; r += 4)
                tma_g4(smem_u32(buf) + s * 16384 + r * 128, &map4, 0, HROW(r), HROW(r + 1), HROW(r + 2), HROW(r + 3), &bar[s]);
        }
        for (int it = iters - S; it < iters; ++it) mbar_wait(&bar[it % S], (it / S) & 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}
__global__ void ldgsts_kernel(const uint16_t* src, const int* rows, int nrows_total, int iters, int W, long long* cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[S];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) mbar_init(&full[s], 32 * W); fence_mbar_init(); }
    __syncthreads();
    long long t0 = clock64();
    if (warp < W) {
        const int sub = lane & 7, rsub = lane >> 3;
        for (int it = 0; it < iters; ++it) {
            const int s = it % S;
            if (it >= S) mbar_wait(&full[s], ((it / S) - 1) & 1);
            const unsigned base = (blockIdx.x * 977u + it * 128u);
            for (int r = 4 * warp + rsub; r < 128; r += 4 * W) {
                const int q = HROW(r);
                cp_async16(smem_u32(buf) + s * 16384 + r * 128 + ((sub ^ (r & 7)) << 4), src + (int64_t)q * 64 + sub * 8, true);
            }
            cpasync_arrive_noinc(&full[s]);
        }
        for (int it = iters - S; it < iters; ++it) mbar_wait(&full[it % S], (it / S) & 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}
int main() {
    const int R = 1 << 20, C = 64;   // 128 MB source (> L2 would be 256 MB; use 16M rows? keep L2-resident like Q)
    const int RQ = 131072;           // 16 MB of distinct rows (L2 resident, like C2's Q)
    uint16_t* d; cudaMalloc(&d, (size_t)R * C * 2); cudaMemset(d, 0, (size_t)R * C * 2);
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)fn;
    CUtensorMap m4;
    cuuint64_t dims[2] = {C, (cuuint64_t)R}, strides[1] = {C * 2};
    cuuint32_t box4[2] = {64, 1}, es[2] = {1, 1};
    enc(&m4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box4, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int NR = 1 << 20;
    std::vector<int> rows(NR);
    unsigned x = 12345;
    for (int i = 0; i < NR; ++i) { x = x * 1664525u + 1013904223u; rows[i] = (x >> 8) % RQ; }
    int* drows; cudaMalloc(&drows, NR * 4); cudaMemcpy(drows, rows.data(), NR * 4, cudaMemcpyHostToDevice);
    long long* dc; cudaMalloc(&dc, 148 * 8);
    std::vector<long long> hc(148);
    const int iters = 400;
    cudaFuncSetAttribute(g4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, S * 16384 + 1024);
    cudaFuncSetAttribute(ldgsts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, S * 16384 + 1024);
    for (int rep = 0; rep < 2; ++rep) {
        g4_kernel<<<148, 32, S * 16384 + 1024>>>(m4, drows, NR, iters, dc);
        cudaDeviceSynchronize();
        cudaMemcpy(hc.data(), dc, 148 * 8, cudaMemcpyDeviceToHost);
        double mx = 0; for (auto c : hc) mx = c > mx ? c : mx;
        printf("gather4 (1 lane, %d in flight): %.1f B/clk/SM  (%.0f clk per 16 KB)  err=%s\n", S, iters * 16384.0 / mx, mx / iters, cudaGetErrorString(cudaGetLastError()));
        for (int W : {1, 2, 3, 4, 6, 8}) {
            ldgsts_kernel<<<148, 32 * W, S * 16384 + 1024>>>(d, drows, NR, iters, W, dc);
            cudaDeviceSynchronize();
            cudaMemcpy(hc.data(), dc, 148 * 8, cudaMemcpyDeviceToHost);
            mx = 0; for (auto c : hc) mx = c > mx ? c : mx;
            printf("ldgsts %d warps (%d in flight): %.1f B/clk/SM  (%.0f clk per 16 KB)  err=%s\n", W, S, iters * 16384.0 / mx, mx / iters, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
