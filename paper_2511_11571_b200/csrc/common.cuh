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
// every exported entry point starts by clearing the previous call's message
void clear_last_error();
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

// 8 consecutive elements (bf16: one 16-B load; fp32: two) as fp32; the
// fp32 forms serve numpy f32/f64 callers, whose Q / K are routed unrounded
MOBA_DEV void ld8f(const __nv_bfloat16* p, float (&x)[8]) {
    const uint4 raw = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t u[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const float2 f = unpack_bf16(u[c]);
        x[2 * c] = f.x;
        x[2 * c + 1] = f.y;
    }
}
MOBA_DEV void ld8f(const float* p, float (&x)[8]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
    x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
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
