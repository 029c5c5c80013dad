// Library-level C ABI helpers: version, status strings, error capture.
#include <cstdio>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace moba {

static thread_local char g_last_error[512] = "";

void set_last_error(const char* msg) {
    std::snprintf(g_last_error, sizeof(g_last_error), "%s", msg);
}

void clear_last_error() { g_last_error[0] = '\0'; }

static unsigned long long g_launches = 0;

int check_launch(const char* what, int n) {
    g_launches += (unsigned long long)n;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        char buf[512];
        std::snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
        set_last_error(buf);
        return MOBA_ERR_CUDA;
    }
    return MOBA_OK;
}

// ---------------------------------------------------------------- stage timing
static const char* kSlotNames[T_NUM_SLOTS] = {"centroid", "route", "varlen", "fwd", "combine",
                                              "bwd_pre", "bwd", "bwd_post", "conv_bwd"};
static bool g_timing = false;
struct EvPair {
    cudaEvent_t a, b;
};
static std::vector<EvPair> g_free;
static std::vector<EvPair> g_pending[T_NUM_SLOTS];
static double g_ms[T_NUM_SLOTS];
static long long g_count[T_NUM_SLOTS];

StageTimer::StageTimer(int s, cudaStream_t st) : slot(s), stream(st), ev(nullptr) {
    if (!g_timing) return;
    EvPair p;
    if (g_free.empty()) {
        cudaEventCreate(&p.a);
        cudaEventCreate(&p.b);
    } else {
        p = g_free.back();
        g_free.pop_back();
    }
    cudaEventRecord(p.a, stream);
    g_pending[slot].push_back(p);
    ev = &g_pending[slot].back();
}

StageTimer::~StageTimer() {
    if (!g_timing || ev == nullptr) return;
    cudaEventRecord(g_pending[slot].back().b, stream);
}

static void drain() {
    for (int s = 0; s < T_NUM_SLOTS; ++s) {
        for (EvPair& p : g_pending[s]) {
            cudaEventSynchronize(p.b);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, p.a, p.b);
            g_ms[s] += ms;
            g_count[s] += 1;
            g_free.push_back(p);
        }
        g_pending[s].clear();
    }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint32_t cols, uint32_t box_rows) {
    static EncodeTiledFn enc = nullptr;
    if (enc == nullptr) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || fn == nullptr) {
            set_last_error("cuTensorMapEncodeTiled unavailable");
            return false;
        }
        enc = (EncodeTiledFn)fn;
    }
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        char buf[96];
        std::snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (%d)", (int)r);
        set_last_error(buf);
        return false;
    }
    return true;
}

// bf16 [heads, rows, cols] with an SW128 box {64, box_rows, 1}: rows past a
// head's end are zero filled instead of reading the next head
bool make_tmap_bf16_3d(CUtensorMap* map, const void* base, uint64_t heads, uint64_t rows, uint32_t cols,
                       uint32_t box_rows) {
    CUtensorMap probe;
    if (!make_tmap_bf16(&probe, base, rows, cols, box_rows)) return false;   // resolves the driver entry point
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || fn == nullptr)
        return false;
    EncodeTiledFn enc = (EncodeTiledFn)fn;
    cuuint64_t dims[3] = {cols, rows, heads};
    cuuint64_t strides[2] = {(cuuint64_t)cols * 2, (cuuint64_t)cols * 2 * rows};
    cuuint32_t box[3] = {64, box_rows, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        char buf[96];
        std::snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled (3-D) failed (%d)", (int)r);
        set_last_error(buf);
        return false;
    }
    return true;
}

// bf16 [outer][mid][cols] with an SW128 box {64, box_mid, box_outer}
bool make_tmap_bf16_3d_box(CUtensorMap* map, const void* base, uint64_t outer, uint64_t mid, uint32_t cols,
                           uint32_t box_mid, uint32_t box_outer) {
    CUtensorMap probe;
    if (!make_tmap_bf16(&probe, base, outer * mid, cols, 1)) return false;   // resolves the driver entry point
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || fn == nullptr)
        return false;
    EncodeTiledFn enc = (EncodeTiledFn)fn;
    cuuint64_t dims[3] = {cols, mid, outer};
    cuuint64_t strides[2] = {(cuuint64_t)cols * 2, (cuuint64_t)cols * 2 * mid};
    cuuint32_t box[3] = {64, box_mid, box_outer};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        char buf[96];
        std::snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled (3-D box) failed (%d)", (int)r);
        set_last_error(buf);
        return false;
    }
    return true;
}

}  // namespace moba

extern "C" const char* moba_version(void) { return "moba_b200 0.1.0 sm_100a"; }

extern "C" const char* moba_last_error(void) { return moba::g_last_error; }

extern "C" const char* moba_status_string(int status) {
    switch (status) {
        case MOBA_OK: return "ok";
        case MOBA_ERR_SHAPE: return "shape error";
        case MOBA_ERR_CONFIG: return "config error";
        case MOBA_ERR_PLAN: return "plan validation error";
        case MOBA_ERR_CUDA: return "CUDA error";
        case MOBA_ERR_UNSUPPORTED: return "unsupported shape for the compiled kernels";
        case MOBA_ERR_WORKSPACE: return "workspace too small";
        default: return "unknown status";
    }
}

extern "C" unsigned long long moba_launch_count(void) { return moba::g_launches; }

extern "C" void moba_timing_enable(int on) {
    moba::drain();
    moba::g_timing = on != 0;
}

extern "C" int moba_timing_enabled(void) { return moba::g_timing ? 1 : 0; }

extern "C" void moba_timing_reset(void) {
    moba::drain();
    for (int s = 0; s < moba::T_NUM_SLOTS; ++s) {
        moba::g_ms[s] = 0.0;
        moba::g_count[s] = 0;
    }
}

extern "C" int moba_timing_read(const char* stage, double* total_ms, long long* launches) {
    moba::drain();
    for (int s = 0; s < moba::T_NUM_SLOTS; ++s) {
        if (std::strcmp(stage, moba::kSlotNames[s]) == 0) {
            *total_ms = moba::g_ms[s];
            *launches = moba::g_count[s];
            return MOBA_OK;
        }
    }
    return MOBA_ERR_CONFIG;
}
