// Microbenchmark: tcgen05.ld (32x32b.x32) throughput per SM, mbarrier round trip.
#include "../../paper_2511_11571_b200/csrc/sm100.cuh"
#include <cstdio>
using namespace moba;
using namespace moba::sm100;

__global__ void tmem_ld_bench(int iters, int nwarps_active, long long* out, float* sink) {
    __shared__ uint32_t tptr;
    __shared__ uint64_t bar;
    int warp = threadIdx.x / 32;
    if (warp == 0) tmem_alloc(&tptr, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    uint32_t tmem = tptr;
    float acc = 0.f;
    long long t0 = clock64();
    if (warp < nwarps_active) {
        uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
        for (int i = 0; i < iters; ++i) {
            float v[32];
            tmem_ld32(tmem + lane_off + (i & 7) * 32 + (warp >> 2) * 256 % 512, v);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 32; ++k) acc += v[k];
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 12345.f) sink[threadIdx.x] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
    long long* d_out; float* sink;
    cudaMalloc(&d_out, 148 * 8); cudaMalloc(&sink, 4096);
    for (int nw : {1, 4, 8, 16}) {
        int iters = 4096;
        tmem_ld_bench<<<148, 512>>>(iters, nw, d_out, sink);
        cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
        double bytes = (double)iters * nw * 32 * 32 * 4;
        printf("warps %2d: %lld cycles, %.1f B/clk/SM (tcgen05.ld 32x32b.x32 + wait)\n", nw, h[0], bytes / h[0]);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
