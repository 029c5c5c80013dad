// Shared device helpers for the sm_100a MoBA kernels.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/moba_b200.h"

#define MOBA_DEV __device__ __forceinline__

namespace moba {

constexpr int kNumSMs = 148;

// ---------------------------------------------------------------- status
void set_last_error(const char* msg);
// checks cudaGetLastError after `n` kernel launches and counts them
int check_launch(const char* what, int n = 1);

// Optional per-stage CUDA-event timing (moba_timing_*), off by default.
enum TimerSlot {
    T_CENTROID = 0, T_ROUTE, T_VARLEN, T_FWD, T_COMBINE, T_BWD_PRE, T_BWD, T_BWD_POST, T_CONV_BWD, T_NUM_SLOTS
};
struct StageTimer {
    StageTimer(int slot, cudaStream_t s);
    ~StageTimer();
    int slot;
    cudaStream_t stream;
    void* ev;
};

// ---------------------------------------------------------------- math
MOBA_DEV float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 2^x for x <= 0 on the FMA/ALU pipes (MUFU offload, as FlashAttention-4):
// j = round(x) via the 1.5*2^23 magic add (no F2I / FRND, which would use the
// same XU pipe as MUFU), f = x - j in [-0.5, 0.5], 2^f by a degree-3
// relative-minimax polynomial (max rel. error 7.7e-5, far below bf16's
// 2^-9), 2^j added to the exponent field. x is clamped at -126.
MOBA_DEV float poly_exp2(float x) {
    x = fmaxf(x, -126.f);
    const float t = x + 12582912.0f;            // low mantissa bits = round(x)
    const float f = x - (t - 12582912.0f);
    float p = fmaf(0.05508876707445847f, f, 0.24260465620999191f);
    p = fmaf(p, f, 0.6932762833525732f);
    p = fmaf(p, f, 0.9999289048020072f);
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// packed fp32x2 arithmetic (sm_100: one FFMA2 / FADD2 for two lanes of data)
MOBA_DEV void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1, float c0, float c1) {
    asm("{\n\t.reg .b64 a, b, c, d;\n\t"
        "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\tmov.b64 c, {%6, %7};\n\t"
        "fma.rn.f32x2 d, a, b, c;\n\tmov.b64 {%0, %1}, d;\n\t}\n"
        : "=f"(d0), "=f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
MOBA_DEV void fadd2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
    asm("{\n\t.reg .b64 a, b, d;\n\t"
        "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
        "add.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}\n"
        : "=f"(d0), "=f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

MOBA_DEV uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

MOBA_DEV float2 unpack_bf16(uint32_t v) {
    __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&v);
    return __bfloat1622float2(h);
}

// ---------------------------------------------------------------- smem / async copy
MOBA_DEV uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// explicit shared-state-space accesses (pointers derived from an aligned
// dynamic-smem base lose their address space; these keep LDS/STS)
MOBA_DEV void sts128(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
MOBA_DEV void sts32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.b32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}
MOBA_DEV float4 lds128f(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}
MOBA_DEV int4 lds128i(uint32_t addr) {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];\n" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
MOBA_DEV int lds32i(uint32_t addr) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1];\n" : "=r"(v) : "r"(addr));
    return v;
}

MOBA_DEV void cp_async16(uint32_t dst, const void* src, bool pred = true) {
    int sz = pred ? 16 : 0;  // src-size 0 => zero fill
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(sz));
}
MOBA_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
MOBA_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---------------------------------------------------------------- legacy tensor-core path
MOBA_DEV void ldmatrix_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
MOBA_DEV void ldmatrix_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
// D = A(16x16, row) * B(16x8, col) + D, bf16 inputs, fp32 accumulate.
MOBA_DEV void mma_bf16_16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// fp32 vector reduction into global memory (no return value).
MOBA_DEV void red_add_f32x2(float* addr, float a, float b) {
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};\n" ::"l"(addr), "f"(a), "f"(b) : "memory");
}
MOBA_DEV void red_add_f32x4(float* addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"l"(addr), "f"(a), "f"(b), "f"(c),
                 "f"(d)
                 : "memory");
}

// Row-major bf16 tile with `kRowBytes` bytes per row, 16-byte chunks XOR
// swizzled by (row & 7) so ldmatrix row fetches hit 8 distinct bank groups.
template <int kRowBytes>
MOBA_DEV uint32_t swz(int row, int chunk) {
    return row * kRowBytes + ((chunk ^ (row & 7)) << 4);
}

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

MOBA_DEV int warp_id() { return threadIdx.x >> 5; }
MOBA_DEV int lane_id() { return threadIdx.x & 31; }

template <typename T>
MOBA_DEV T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
template <typename T>
MOBA_DEV T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// bf16 [rows, cols] row-major tensor map with an SW128 box {64, box_rows}
bool make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint32_t cols, uint32_t box_rows);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace moba
