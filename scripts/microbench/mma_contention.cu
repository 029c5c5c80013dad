// Microbenchmark: does concurrent TMEM / shared-memory traffic from other
// warps slow the backward's per-tile MMA mix (8x TS dV, 8x TS dK, 8x SS dQ)?
// LOAD 0: MMA warp alone; 1: 8 warps loop tcgen05.ld x32 (+wait) on other
// columns; 2: 8 warps loop 16-B shared-memory stores + loads; 3: both.
#include "../../paper_2511_11571_b200/csrc/sm100.cuh"
#include <cstdio>
using namespace moba;
using namespace moba::sm100;

template <int LOAD>
__global__ void mix(int reps, long long* out, float* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tptr;
    __shared__ uint64_t bar;
    __shared__ volatile int done;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0) tmem_alloc(&tptr, 512);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); done = 0; }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tptr;
    const uint32_t sa = smem_u32(sm), sb = sa + 32768;
    if (warp == 0) {
        const uint32_t id_kd = idesc_bf16(128, 64, false, true), id_qd = idesc_bf16(128, 64, true, true);
        long long t0 = clock64();
        if (lane == 0) {
            for (int r = 0; r < reps; ++r) {
                for (int kk = 0; kk < 8; ++kk) {
                    umma_bf16_ts(tmem + 384, tmem + 8 * kk, desc_mnmajor(sb, kk * 16, 128 * 128), id_kd, kk > 0);
                    umma_bf16_ts(tmem + 448, tmem + 256 + 8 * kk, desc_mnmajor(sb, kk * 16, 128 * 128), id_kd, kk > 0);
                }
                for (int kk = 0; kk < 8; ++kk)
                    umma_bf16(tmem + 64, desc_mnmajor(sa, kk * 16, 128 * 128), desc_mnmajor(sb, kk * 16, 128 * 128),
                              id_qd, kk > 0);
            }
            umma_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (lane == 0 && blockIdx.x == 0) out[0] = t1 - t0;
        if (lane == 0) done = 1;
    } else if (warp >= 4 && warp < 12) {
        const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
        float acc = 0.f;
        int it = 0;
        while (!done) {
            if (LOAD & 1) {
                float v[32];
                tmem_ld32(tmem + lane_off + 128 + 32 * ((it + warp) & 3), v);
                tmem_ld_wait();
                acc += v[lane & 31];
            }
            if (LOAD & 2) {
                const uint32_t o = ((uint32_t)(warp * 32 + lane) * 16u + (uint32_t)it * 4096u) & 65535u;
                sts128(sa + 65536 + o, make_uint4(it, it, it, it));
                acc += __int_as_float(lds32i(sa + 65536 + ((o + 4096u) & 65535u)));
            }
            ++it;
        }
        if (acc == 12345.f) sink[0] = acc;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
    long long* d; cudaMalloc(&d, 16);
    float* sink; cudaMalloc(&sink, 4);
    const char* names[] = {"alone", "+ LDTM x32 loops (8 warps)", "+ smem st/ld loops (8 warps)", "+ both"};
    for (int load = 0; load < 4; ++load) {
        auto k = load == 0 ? mix<0> : load == 1 ? mix<1> : load == 2 ? mix<2> : mix<3>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072 + 1024);
        long long h = 0;
        for (int rep = 0; rep < 3; ++rep) {
            k<<<1, 512, 131072 + 1024>>>(40, d, sink);
            cudaDeviceSynchronize();
        }
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("bwd MMA mix (40 x 24 MMAs) %-30s %8lld clk  %.1f clk/MMA  %s\n", names[load], h, h / 960.0,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
