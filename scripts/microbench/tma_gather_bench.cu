// Microbenchmark / correctness probe: TMA 2D row loads vs tile::gather4 (SW128).
#include "../../paper_2511_11571_b200/csrc/sm100.cuh"
#include <cuda.h>
#include <cstdio>
#include <vector>
using namespace moba;
using namespace moba::sm100;

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ void tma_row(uint32_t dst, const CUtensorMap* map, int c0, int row, uint64_t* bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 :: "r"(dst), "l"(map), "r"(c0), "r"(row), "r"(smem_u32(bar)) : "memory");
}
__device__ void tma_g4(uint32_t dst, const CUtensorMap* map, int c0, int r0, int r1, int r2, int r3, uint64_t* bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                 :: "r"(dst), "l"(map), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar)) : "memory");
}

__global__ void probe(const __grid_constant__ CUtensorMap map1, const __grid_constant__ CUtensorMap map4, int mode,
                      const int* rows, int nrows, int iters, uint16_t* out, long long* cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (threadIdx.x == 0) {
            mbar_expect_tx(&bar, nrows * 128);
        }
        __syncwarp();
        if (threadIdx.x < 32) {
            if (mode == 0) {
                for (int r = threadIdx.x; r < nrows; r += 32) tma_row(smem_u32(buf) + r * 128, &map1, 0, rows[r], &bar);
            } else {
                for (int r = threadIdx.x * 4; r < nrows; r += 128)
                    tma_g4(smem_u32(buf) + r * 128, &map4, 0, rows[r], rows[r + 1], rows[r + 2], rows[r + 3], &bar);
            }
        }
        mbar_wait(&bar, it & 1);
    }
    long long t1 = clock64();
    __syncthreads();
    if (blockIdx.x == 0) {
        for (int e = threadIdx.x; e < nrows * 64; e += blockDim.x) {
            int r = e / 64, c = e % 64;
            out[e] = *(uint16_t*)(buf + sw128_off(r, c, nrows));
        }
        if (threadIdx.x == 0) cyc[0] = t1 - t0;
    }
}

int main() {
    const int R = 65536, C = 64;
    std::vector<uint16_t> h(R * C);
    for (int i = 0; i < R * C; ++i) h[i] = (uint16_t)(i * 7 + 3);
    uint16_t* d; cudaMalloc(&d, h.size() * 2); cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)fn;
    CUtensorMap m1, m4a, m4b;
    cuuint64_t dims[2] = {C, R}, strides[1] = {C * 2};
    cuuint32_t box1[2] = {64, 1}, box4[2] = {64, 4}, es[2] = {1, 1};
    printf("enc1 %d\n", enc(&m1, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box1, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
    printf("enc4 %d\n", enc(&m4a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box4, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
    const int NR = 128;
    std::vector<int> rows(NR);
    for (int i = 0; i < NR; ++i) rows[i] = (i * 7919 + 13) % R;
    int* drows; cudaMalloc(&drows, NR * 4); cudaMemcpy(drows, rows.data(), NR * 4, cudaMemcpyHostToDevice);
    uint16_t* dout; cudaMalloc(&dout, NR * 64 * 2);
    long long* dc; cudaMalloc(&dc, 8);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    struct { const char* name; int mode; CUtensorMap* m4; } cases[] = {{"row-2D", 0, &m1}, {"gather4 box{64,1}", 1, &m1}, {"gather4 box{64,4}", 1, &m4a}};
    for (auto& cs : cases) {
        cudaMemset(dout, 0, NR * 128);
        probe<<<148, 128, 40 * 1024>>>(m1, *cs.m4, cs.mode, drows, NR, 200, dout, dc);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<uint16_t> o(NR * 64); long long cyc = 0;
        cudaMemcpy(o.data(), dout, NR * 128, cudaMemcpyDeviceToHost); cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int r = 0; r < NR; ++r) for (int c = 0; c < 64; ++c) if (o[r * 64 + c] != h[rows[r] * 64 + c]) ++bad;
        printf("%-20s err=%s bad=%d cycles/128rows=%.0f (%.1f B/clk/SM)\n", cs.name, cudaGetErrorString(e), bad, cyc / 200.0, 128 * 128 / (cyc / 200.0));
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
