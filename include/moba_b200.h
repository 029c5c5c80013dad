/*
 * moba_b200.h — C ABI of the B200-native MoBA attention hot path.
 *
 * This is the drop-in boundary for the reference's MoBA attention call
 * (/root/reference/pkg/src/moba, cited as src/<file>:<line>). Every entry
 * point below replaces one numpy stage of the reference; the Python host
 * package `paper_2511_11571_b200` binds them with ctypes and mirrors the
 * reference's operator API on top (same names, argument meaning, errors).
 *
 * Conventions
 *   - plain pointers and sizes; no framework types. All tensor pointers are
 *     DEVICE pointers (CUDA global memory), caller-allocated.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *   - every call is asynchronous on `stream` unless stated otherwise and
 *     returns a moba_status (0 = OK). Status codes map to the reference's
 *     exception classes (src/core.py:17-38): SHAPE -> ShapeError,
 *     CONFIG -> ConfigError, PLAN -> PlanValidationError.
 *   - layouts: a "head" is one independent (batch, head) pair; `bh` heads are
 *     stored back to back. Q/K/V/O/dO/dQ/dK/dV are bf16 [bh, n_tokens,
 *     head_dim] row-major; head_dim is 64 or 128 (callers with a smaller d
 *     zero-pad channels and pass the true softmax scale 1/sqrt(d)).
 *   - routing plan (RoutingPlan, src/core.py:229-251), per head:
 *       topk    int32 [n_tokens, width]   width = top_k + 1, rows ascending,
 *                                          -1 tail (src/router.py:116-119)
 *       counts  int32 [n_blocks]           queries attending block j
 *       offsets int32 [n_blocks]           exclusive prefix sum of counts
 *       flat    int32 [n_tokens * width]   block j's attending queries at
 *                                          flat[offsets[j] .. +counts[j]),
 *                                          strictly ascending
 *       row_pos int32 [n_tokens, width]    inverse map: flat position of
 *                                          (query, slot), -1 for sentinels
 *     head h's arrays start at h * (their per-head size); offsets are
 *     head-local.
 */
#ifndef MOBA_B200_H
#define MOBA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MOBA_OK = 0,
    MOBA_ERR_SHAPE = 1,        /* ShapeError            */
    MOBA_ERR_CONFIG = 2,       /* ConfigError           */
    MOBA_ERR_PLAN = 3,         /* PlanValidationError   */
    MOBA_ERR_CUDA = 4,         /* CUDA launch / runtime */
    MOBA_ERR_UNSUPPORTED = 5,  /* shape outside the compiled kernels */
    MOBA_ERR_WORKSPACE = 6     /* workspace too small   */
} moba_status;

/* Routing mode for moba_route. */
#define MOBA_ROUTE_FP32 0      /* exact fp32 FFMA scores (parity mode)       */
#define MOBA_ROUTE_TC   1      /* tensor-core scores, centroid split hi/lo   */

/* Library version and the status string for an error code. */
const char* moba_version(void);
const char* moba_status_string(int status);
/* Last CUDA error text recorded by the library (thread-local). */
const char* moba_last_error(void);

/*
 * Stage 1 — centroids (+ optional causal key short-conv).
 * Replaces compute_centroids (src/router.py:32-46) and key_conv_forward
 * (src/keyconv.py:70-78):
 *   a_t  = sum_{l<width} W[l] * K[t-l]   (zero left pad)
 *   K'_t = K_t + a_t * sigmoid(a_t)      (written as bf16 to k_conv_out)
 *   centroid_j = mean over the (ragged) block of K' (fp32, unrounded K')
 * conv_w: fp32 [conv_width, head_dim] device pointer, or NULL with
 * conv_width = 0 (then k_conv_out may be NULL). centroids: fp32
 * [bh, n_blocks, head_dim].
 */
int moba_centroids(const void* k, const float* conv_w, int conv_width,
                   int64_t bh, int64_t n_tokens, int head_dim, int block_size,
                   void* k_conv_out, float* centroids, void* stream);

/*
 * moba_centroids with fp32 keys (numpy f32 / f64 callers of
 * compute_centroids / key_conv_forward, src/router.py:32-46): the centroids
 * (and the conv's unrounded K') come from the caller's unrounded keys;
 * k_conv_out is still bf16 (the attention operand).
 */
int moba_centroids_f32(const float* k, const float* conv_w, int conv_width,
                       int64_t bh, int64_t n_tokens, int head_dim, int block_size,
                       void* k_conv_out, float* centroids, void* stream);

/* Workspace bytes needed by moba_route / moba_varlen. The varlen chunk
 * geometry depends on bh and the row width, so pass the call's top_k (for
 * moba_varlen: width - 1); a smaller workspace returns MOBA_ERR_WORKSPACE. */
size_t moba_route_workspace_size(int64_t bh, int64_t n_tokens, int block_size, int top_k);

/*
 * Stages 2+3 — tiled top-k routing and the varlen plan.
 * Replaces select_topk (src/router.py:49-120) + build_varlen
 * (src/router.py:123-154), i.e. build_plan after the centroids
 * (src/router.py:157-161). Scores are the UNSCALED q . centroid
 * (src/attention.py:312); only strictly-past blocks compete; ties go to the
 * lower block index; the own block is always added. Never materialises the
 * [n_tokens, n_blocks] score matrix.
 */
int moba_route(const void* q, const float* centroids,
               int64_t bh, int64_t n_tokens, int head_dim, int block_size,
               int top_k, int mode,
               int32_t* topk, int32_t* counts, int32_t* offsets,
               int32_t* flat, int32_t* row_pos,
               void* workspace, size_t workspace_bytes, void* stream);

/*
 * moba_route_gqa in fp32 routing mode with fp32 queries [bh, n_tokens,
 * head_dim] (numpy f32 / f64 callers of select_topk, src/router.py:49-120):
 * scores are exact fp32 products of the caller's unrounded q and the fp32
 * centroids, so routing is not perturbed by rounding Q to bf16.
 */
int moba_route_f32(const float* q, const float* centroids, int64_t bh, int kv_group,
                   int64_t n_tokens, int head_dim, int block_size, int top_k,
                   int32_t* topk, int32_t* counts, int32_t* offsets, int32_t* flat, int32_t* row_pos,
                   void* workspace, size_t workspace_bytes, void* stream);

/*
 * Stage 3 alone — varlen layout from a caller-supplied index matrix
 * (build_varlen, src/router.py:123-154). width = columns of topk.
 * Entries outside [-1, n_blocks) -> MOBA_ERR_PLAN (synchronous check).
 */
int moba_varlen(const int32_t* topk, int64_t bh, int64_t n_tokens, int width,
                int block_size,
                int32_t* counts, int32_t* offsets, int32_t* flat, int32_t* row_pos,
                void* workspace, size_t workspace_bytes, void* stream);

/*
 * row_pos for a caller-built plan: for every (query, slot) the position of
 * the query inside block topk[query][slot]'s ascending slice (binary
 * search), -1 for sentinels. Plans from moba_route/moba_varlen already carry
 * it. Used by moba_fwd's combine step.
 */
int moba_plan_row_pos(const int32_t* topk, const int32_t* counts, const int32_t* offsets,
                      const int32_t* flat, int64_t bh, int64_t n_tokens, int width,
                      int block_size, int32_t* row_pos, void* stream);

/*
 * validate_plan (src/core.py:254-296) on device. SYNCHRONOUS (reads back a
 * flag word). Returns MOBA_ERR_PLAN if any invariant fails: range,
 * causality (block <= query / B), per-row uniqueness, offsets = exclusive
 * prefix sum, sum(counts) = non-sentinel entries, slices strictly
 * ascending with queries in [jB, N).
 */
int moba_validate_plan(const int32_t* topk, const int32_t* counts,
                       const int32_t* offsets, const int32_t* flat,
                       int64_t bh, int64_t n_tokens, int width, int block_size,
                       void* workspace, size_t workspace_bytes, void* stream);

/* Workspace bytes for moba_fwd / moba_bwd. */
size_t moba_fwd_workspace_size(int64_t bh, int64_t n_tokens, int head_dim,
                               int block_size, int width);
size_t moba_bwd_workspace_size(int64_t bh, int64_t n_tokens, int head_dim,
                               int block_size, int width, int deterministic);

/*
 * Forward — gather-and-densify (moba_forward, src/attention.py:147-182;
 * Alg. 1 of the paper). Per (key block, 128 gathered queries) the kernel
 * computes S = Q K_j^T * scale, the causal mask key > query
 * (src/attention.py:127-133), softmax and P V_j densely, writes a
 * per-(query, block) partial, and a combine kernel merges each query's
 * partials into O (bf16) and LSE (fp32, natural log; src/attention.py:70-74).
 */
int moba_fwd(const void* q, const void* k, const void* v,
             int64_t bh, int64_t n_tokens, int head_dim, int block_size, int width,
             const int32_t* counts, const int32_t* offsets,
             const int32_t* flat, const int32_t* row_pos,
             float softmax_scale,
             void* out, float* lse,
             void* workspace, size_t workspace_bytes, void* stream);

/*
 * Backward — recomputation (moba_backward, src/attention.py:239-302;
 * Alg. 5). D = rowsum(dO * O) (src/attention.py:266); per key block the
 * kernel gathers the block's queries, recomputes P = exp(S - L), and
 * accumulates dV_j, dK_j on chip and dQ into an fp32 accumulator
 * (src/attention.py:229-234); dQ = accum * scale -> bf16
 * (src/attention.py:299). lse must be finite (src/attention.py:255-259;
 * checked by the host layer).
 * deterministic != 0 mirrors schedule="deterministic" (src/attention.py:
 * 294-297): dQ partials are written per (query, block) and summed in slot
 * order (bitwise repeatable; needs row_pos). deterministic == 0 mirrors
 * schedule="parallel" (src/attention.py:276-293): fp32 vector reductions
 * into one dQ accumulator (order-dependent rounding).
 */
int moba_bwd(const void* q, const void* k, const void* v,
             const void* out, const void* dout, const float* lse,
             int64_t bh, int64_t n_tokens, int head_dim, int block_size, int width,
             const int32_t* counts, const int32_t* offsets, const int32_t* flat,
             const int32_t* row_pos, int deterministic,
             float softmax_scale,
             void* dq, void* dk, void* dv,
             void* workspace, size_t workspace_bytes, void* stream);

/*
 * Grouped-query attention (GQA / MQA). Same operations as
 * moba_route / moba_fwd / moba_bwd with `bh` QUERY heads sharing
 * bh / kv_group K/V heads: query head h reads K, V (and, for routing, the
 * centroids) of K/V head h / kv_group. centroids, k, v, dk, dv are
 * [bh / kv_group, n_tokens, head_dim]; dK / dV are the sums over the
 * kv_group query heads of each K/V head (fixed order). kv_group = 1 is the
 * reference's multi-head case (the plain entry points call these).
 */
int moba_route_gqa(const void* q, const float* centroids, int64_t bh, int kv_group,
                   int64_t n_tokens, int head_dim, int block_size, int top_k, int mode,
                   int32_t* topk, int32_t* counts, int32_t* offsets, int32_t* flat, int32_t* row_pos,
                   void* workspace, size_t workspace_bytes, void* stream);
int moba_fwd_gqa(const void* q, const void* k, const void* v, int64_t bh, int kv_group,
                 int64_t n_tokens, int head_dim, int block_size, int width,
                 const int32_t* counts, const int32_t* offsets, const int32_t* flat, const int32_t* row_pos,
                 float softmax_scale, void* out, float* lse,
                 void* workspace, size_t workspace_bytes, void* stream);
size_t moba_bwd_gqa_workspace_size(int64_t bh, int kv_group, int64_t n_tokens, int head_dim,
                                   int block_size, int width, int deterministic);
int moba_bwd_gqa(const void* q, const void* k, const void* v, const void* out, const void* dout,
                 const float* lse, int64_t bh, int kv_group, int64_t n_tokens, int head_dim,
                 int block_size, int width, const int32_t* counts, const int32_t* offsets,
                 const int32_t* flat, const int32_t* row_pos, int deterministic, float softmax_scale,
                 void* dq, void* dk, void* dv, void* workspace, size_t workspace_bytes, void* stream);

/*
 * Key-conv backward (key_conv_backward, src/keyconv.py:81-104):
 *   g = dK' * silu'(a);  dK = dK' + sum_l W[l] * g_{t+l};  dW[l] = sum_t g_t K_{t-l}
 * k, dk_conv: bf16 [bh, n_tokens, head_dim]; dk: bf16 out; dw: fp32
 * [conv_width, head_dim] summed over heads (one W shared across heads,
 * src/cli.py:255-258). workspace: fp32 partials for the dW reduction.
 */
size_t moba_conv_bwd_workspace_size(int64_t bh, int64_t n_tokens, int head_dim, int conv_width);
int moba_conv_bwd(const void* k, const float* conv_w, int conv_width, const void* dk_conv,
                  int64_t bh, int64_t n_tokens, int head_dim,
                  void* dk, float* dw, void* workspace, size_t workspace_bytes, void* stream);

/*
 * Instrumentation (the reference's OpCounters / perf_counter role,
 * src/core.py:193-226): kernels launched so far, and optional per-stage
 * CUDA-event timing recorded on the launching stream. Stage names:
 * centroid, route, varlen, fwd, combine, bwd_pre, bwd, bwd_post, conv_bwd.
 * moba_timing_read synchronises on the recorded events.
 */
unsigned long long moba_launch_count(void);
void moba_timing_enable(int on);
int moba_timing_enabled(void);
void moba_timing_reset(void);
int moba_timing_read(const char* stage, double* total_ms, long long* launches);

#ifdef __cplusplus
}
#endif
#endif /* MOBA_B200_H */
