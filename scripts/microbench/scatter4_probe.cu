// Probe: semantics of cp.reduce.async.bulk.tensor ... tile::scatter4 on sm_100a
// with an fp32 box {32, 1} and SWIZZLE_128B / NONE. Stages 32 rows x 32 fp32
// (value = 1000 * staged_row + col) in smem, scatters 8 ops of 4 rows
// (op m at smem + 512 m) to global rows {2m, 2m+16, 2m+32, 2m+48}, prints
// where the values landed.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int SW>   // SW: 0 none, 1 absolute-address SW128 staging
__global__ void probe(const __grid_constant__ CUtensorMap tm) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
    const int r = threadIdx.x;   // staged row 0..31
    for (int c = 0; c < 8; ++c) {
        float v[4];
        for (int u = 0; u < 4; ++u) v[u] = 1000.f * r + 4 * c + u;
        const int pos = SW ? (c ^ (r & 7)) : c;
        float* p = reinterpret_cast<float*>(sm + r * 128 + pos * 16);
        for (int u = 0; u < 4; ++u) p[u] = v[u];
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
    if (r < 8) {
        const int m = r;
        asm volatile(
            "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile::scatter4.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];\n"
            ::"l"(&tm), "r"(0), "r"(2 * m), "r"(2 * m + 16), "r"(2 * m + 32), "r"(2 * m + 48), "r"(base + 512 * m) : "memory");
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    }
}

int main() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)fn;
    float* g;
    cudaMalloc(&g, 64 * 64 * 4);
    for (int sw = 0; sw < 2; ++sw) {
        cudaMemset(g, 0, 64 * 64 * 4);
        CUtensorMap tm;
        cuuint64_t dims[2] = {64, 64};
        cuuint64_t strides[1] = {64 * 4};
        cuuint32_t box[2] = {32, 1};
        cuuint32_t es[2] = {1, 1};
        CUresult rr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (sw) probe<1><<<1, 32, 8192>>>(tm); else probe<0><<<1, 32, 8192>>>(tm);
        cudaError_t e = cudaDeviceSynchronize();
        float h[64 * 64];
        cudaMemcpy(h, g, sizeof(h), cudaMemcpyDeviceToHost);
        printf("swizzle=%d encode=%d err=%s\n", sw, (int)rr, cudaGetErrorString(e));
        for (int row : {0, 16, 32, 48, 2, 18, 34, 50, 14, 62, 1}) {
            printf("  g row %2d:", row);
            for (int c : {0, 1, 4, 8, 28, 31, 32}) printf(" %7.0f", h[row * 64 + c]);
            printf("\n");
        }
    }
    return 0;
}
