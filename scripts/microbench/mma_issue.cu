// Microbenchmark: issue cost vs execution time of back-to-back tcgen05.mma
// from one thread (SS and TS forms, N = 64 / 128), with and without the
// warp-uniform elect.sync variant.
#include "../../paper_2511_11571_b200/csrc/sm100.cuh"
#include <cstdio>
using namespace moba;
using namespace moba::sm100;

template <int MODE>   // 0: SS N=128, 1: SS N=64, 2: TS N=64, 3: SS N=64 warp-uniform,
                      // 4: SS N=64 both operands MN-major (the backward's dQ), 5: the backward's
                      // per-tile mix (TS dV, TS dK interleaved, then SS MN-major dQ), n = MMAs
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
        const uint32_t idesc = idesc_bf16(128, (MODE == 0) ? 128 : 64, MODE == 4, MODE == 2 || MODE == 4);
        if (MODE == 5) {
            const uint32_t id_kd = idesc_bf16(128, 64, false, true), id_qd = idesc_bf16(128, 64, true, true);
            if (lane == 0) {
                t0 = clock64();
                for (int i = 0; i < n; i += 24) {
                    for (int kk = 0; kk < 8; ++kk) {
                        umma_bf16_ts(tmem + 384, tmem + 8 * kk, desc_mnmajor(sb, kk * 16, 128 * 128), id_kd, kk > 0);
                        umma_bf16_ts(tmem + 448, tmem + 256 + 8 * kk, desc_mnmajor(sb, kk * 16, 128 * 128), id_kd, kk > 0);
                    }
                    for (int kk = 0; kk < 8; ++kk)
                        umma_bf16(tmem + 64, desc_mnmajor(sa, kk * 16, 128 * 128), desc_mnmajor(sb, kk * 16, 128 * 128),
                                  id_qd, kk > 0);
                }
                umma_commit(&bar);
                t1 = clock64();
            }
        } else if (MODE == 4) {
            if (lane == 0) {
                t0 = clock64();
                for (int i = 0; i < n; ++i)
                    umma_bf16(tmem + 256, desc_mnmajor(sa, (i & 7) * 16, 128 * 128), desc_mnmajor(sb, (i & 7) * 16, 128 * 128),
                              idesc, i > 0);
                umma_commit(&bar);
                t1 = clock64();
            }
        } else if (MODE == 3) {
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
    const char* names[] = {"SS M128 N128 K16", "SS M128 N64 K16", "TS M128 N64 K16", "SS N64 warp-uniform",
                           "SS N64 MN-major A,B", "bwd mix (dV,dK TS; dQ SS)"};
    for (int mode = 0; mode < 6; ++mode) {
        for (int n : {24, 48, 96}) {
            long long h[2] = {0, 0};
            for (int rep = 0; rep < 3; ++rep) {
                auto k = mode == 0 ? mma_issue<0> : mode == 1 ? mma_issue<1> : mode == 2 ? mma_issue<2> : mode == 3 ? mma_issue<3>
                         : mode == 4 ? mma_issue<4> : mma_issue<5>;
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
