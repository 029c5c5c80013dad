// MUFU.EX2 throughput on sm_100a: W warps per SM each issuing chains of
// independent ex2.approx.ftz.f32 (8 per iteration, 4096 iterations);
// clk per warp-instruction per SMSP = (cycles x SMSPs) / (ex2 issued / 32).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a mufu_ex2.cu -o mufu_ex2
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ unsigned pack2(float a, float b) {
    unsigned r;
    asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
    return r;
}

// 0: ex2 only, 1: ex2 + 1 FFMA each, 2: ex2 + one bf16x2 pack per two ex2
// (the forward softmax's mix), 3: bf16x2 packs only
template <int MODE>
__global__ void k(float* out, long long* clk, int iters) {
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = -1.0f / (threadIdx.x + i + 1);
    __syncthreads();
    const long long t0 = clock64();
    unsigned acc = 0;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 3) {
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
                acc ^= pack2(a[i], a[i + 1]);
                a[i] += 1e-7f;
                a[i + 1] -= 1e-7f;
            }
            continue;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 1) a[i] = fmaf(a[i], 0.999f, -0.001f);
            a[i] = ex2(a[i]) - 1.0f;
        }
        if (MODE == 2) {
#pragma unroll
            for (int i = 0; i < 8; i += 2) acc ^= pack2(a[i], a[i + 1]);
        }
    }
    a[0] += (float)(acc & 1);
    const long long t1 = clock64();
    __syncthreads();
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
    float* out;
    long long* clk;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&clk, 148 * 8);
    const int iters = 4096;
    for (int mode = 0; mode < 4; ++mode)
        for (int warps : {4, 8, 16}) {
            auto launch = [&]() {
                if (mode == 0) k<0><<<148, warps * 32>>>(out, clk, iters);
                else if (mode == 1) k<1><<<148, warps * 32>>>(out, clk, iters);
                else if (mode == 2) k<2><<<148, warps * 32>>>(out, clk, iters);
                else k<3><<<148, warps * 32>>>(out, clk, iters);
            };
            launch();
            cudaDeviceSynchronize();
            launch();
            long long h[148];
            cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
            double c = 0;
            for (int i = 0; i < 148; ++i) c += h[i];
            c /= 148;
            const double instr_per_smsp = (double)iters * 8 * warps / 4;
            const char* nm[4] = {"ex2", "ex2+ffma", "ex2+pack/2", "pack only (per 2 elems)"};
            const double per = mode == 3 ? instr_per_smsp / 2 : instr_per_smsp;
            printf("mode %d (%s) warps/SM %2d: %.2f clk per %s warp-instruction per SMSP\n", mode, nm[mode], warps,
                   c / per, mode == 3 ? "pack" : "ex2");
        }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
