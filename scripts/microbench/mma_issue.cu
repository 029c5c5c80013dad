// Microbenchmark: issue cost vs execution time of back-to-back tcgen05.mma
// from one thread (SS and TS forms, N = 64 / 128), with and without the
// warp-uniform elect.sync variant.
#include "../../paper_2511_11571_b200/csrc/sm100.cuh"
#include <cstdio>
using namespace moba;
using namespace moba::sm100;

template <int MODE>   // 0: SS N=128, 1: SS N=64, 2: TS N=64, 3: SS N=64 warp-uniform
__global__ void mma_issue(int n, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tptr;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0) tmem_alloc(&tptr, 512);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tptr;
    const uint32_t sa = smem_u32(sm), sb = sa + 32768;
    long long t0 = 0, t1 = 0, t2 = 0;
    if (warp == 0) {
        const uint32_t idesc = idesc_bf16(128, (MODE == 0) ? 128 : 64, false, MODE == 2);
        if (MODE == 3) {
            t0 = clock64();
            for (int i = 0; i < n; ++i)
                umma_bf16_w(tmem + 256, desc_kmajor(sa, (i & 3) * 16), desc_kmajor(sb, (i & 3) * 16), idesc, i > 0);
            umma_commit_w(&bar);
            t1 = clock64();
        } else if (lane == 0) {
            t0 = clock64();
            for (int i = 0; i < n; ++i) {
                if (MODE == 2)
                    umma_bf16_ts(tmem + 256, tmem + 8 * (i & 7), desc_mnmajor(sb, (i & 7) * 16, 128 * 128), idesc, i > 0);
                else
                    umma_bf16(tmem + 256, desc_kmajor(sa, (i & 3) * 16), desc_kmajor(sb, (i & 3) * 16), idesc, i > 0);
            }
            umma_commit(&bar);
            t1 = clock64();
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        t2 = clock64();
        if (lane == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
    long long* d; cudaMalloc(&d, 16);
    const char* names[] = {"SS M128 N128 K16", "SS M128 N64 K16", "TS M128 N64 K16", "SS N64 warp-uniform"};
    for (int mode = 0; mode < 4; ++mode) {
        for (int n : {8, 32, 128}) {
            long long h[2] = {0, 0};
            for (int rep = 0; rep < 3; ++rep) {
                auto k = mode == 0 ? mma_issue<0> : mode == 1 ? mma_issue<1> : mode == 2 ? mma_issue<2> : mma_issue<3>;
                cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
                k<<<1, 128, 65536 + 1024>>>(n, d);
                cudaDeviceSynchronize();
            }
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            printf("%-22s n=%4d  issue %6lld clk (%.1f/mma)  complete %6lld clk (%.1f/mma)  %s\n", names[mode], n, h[0],
                   (double)h[0] / n, h[1], (double)h[1] / n, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
