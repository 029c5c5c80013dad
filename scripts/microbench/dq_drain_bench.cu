// Throughput of the ways a CTA can add fp32 rows into an L2-resident
// accumulator (the backward's dQ drain): per-row cp.reduce.async.bulk
// (256 B / 512 B ops, 16 or 32 issuing lanes per warp), red.global.add.v4.f32
// from registers, and plain cp.async.bulk stores (no reduction) for
// comparison. Rows are random within a 48 MB buffer, as gathered queries are.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I ../../paper_2511_11571_b200/csrc dq_drain_bench.cu -o dq_drain_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"
#include "sm100.cuh"

using namespace moba;
using namespace moba::sm100;

constexpr int kRows = 48 << 20 >> 8;      // 48 MB of 256-B rows
constexpr int kTiles = 200;               // tiles per CTA
constexpr int kRowsPerTile = 128;

__device__ __forceinline__ uint32_t hash(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16;
    return x;
}

// mode 0: bulk reduce 256 B per row, lanes 0-15 then 16-31 issue (the kernel's scheme)
// mode 1: bulk reduce 256 B per row, all 32 lanes issue at once
// mode 2: red.global.add.v4.f32 from registers (16 lanes x 16 B per row, 2 rows per instruction)
// mode 3: bulk store 256 B per row (no reduction)
// mode 4: bulk reduce 512 B (two adjacent rows merged)
template <int MODE>
__global__ void __launch_bounds__(128) drain(float* acc) {
    __shared__ __align__(128) float stg[128][64];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = threadIdx.x;
    for (int i = 0; i < 64; ++i) stg[row][i] = 1.0f;
    __syncthreads();
    fence_proxy_async_smem();
    for (int t = 0; t < kTiles; ++t) {
        const uint32_t r = hash(blockIdx.x * 7919u + t * 131u + row) % (MODE == 4 ? kRows / 2 : kRows);
        if (MODE == 0) {
            for (int rr = 0; rr < 2; ++rr) {
                bulk_wait_read0();
                __syncwarp();
                if ((lane >> 4) == rr) {
                    bulk_reduce_add_f32(acc + (size_t)r * 64, smem_u32(&stg[row][0]), 256);
                    bulk_commit();
                }
            }
        } else if (MODE == 1) {
            bulk_wait_read0();
            bulk_reduce_add_f32(acc + (size_t)r * 64, smem_u32(&stg[row][0]), 256);
            bulk_commit();
        } else if (MODE == 2) {
            float* dst = acc + (size_t)r * 64;
#pragma unroll
            for (int i = 0; i < 64; i += 4) red_add_f32x4(dst + i, 1.f, 1.f, 1.f, 1.f);
        } else if (MODE == 3) {
            bulk_wait_read0();
            bulk_store(acc + (size_t)r * 64, smem_u32(&stg[row][0]), 256);
            bulk_commit();
        } else {
            bulk_wait_read0();
            if (row < 64) {
                bulk_reduce_add_f32(acc + (size_t)r * 128, smem_u32(&stg[2 * row][0]), 512);
                bulk_commit();
            }
        }
        (void)warp;
    }
    bulk_wait0();
}

template <int MODE>
static void run(float* acc, const char* name, int per_sm = 4) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    drain<MODE><<<148 * per_sm, 128>>>(acc);
    cudaEventRecord(a);
    drain<MODE><<<148 * per_sm, 128>>>(acc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = 148.0 * per_sm * kTiles * kRowsPerTile * 256;
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double per_sm_clk = bytes / (ms * 1e-3) / 148 / (clk * 1e3);
    printf("%-44s x%d/SM %8.3f ms  %7.2f TB/s  %6.1f B/clk/SM  (%.0f clk per 128-row tile per CTA)\n", name, per_sm,
           ms, bytes / (ms * 1e-3) / 1e12, per_sm_clk, 128 * 256 / per_sm_clk * per_sm);
}

int main() {
    float* acc;
    cudaMalloc(&acc, (size_t)kRows * 256);
    cudaMemset(acc, 0, (size_t)kRows * 256);
    run<0>(acc, "bulk reduce 256 B, 16 lanes x 2 rounds");
    run<1>(acc, "bulk reduce 256 B, 32 lanes");
    run<4>(acc, "bulk reduce 512 B (2 rows merged)");
    run<2>(acc, "red.global.add.v4.f32 from registers");
    run<3>(acc, "bulk store 256 B (no reduction)");
    run<0>(acc, "bulk reduce 256 B, 16 lanes x 2 rounds", 1);
    run<1>(acc, "bulk reduce 256 B, 32 lanes", 1);
    run<3>(acc, "bulk store 256 B (no reduction)", 1);
    run<0>(acc, "bulk reduce 256 B, 16 lanes x 2 rounds", 2);
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
