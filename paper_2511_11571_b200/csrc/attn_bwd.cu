// Backward: key-block-major recomputation (moba_backward,
// src/attention.py:239-302; paper Alg. 5).
//
//   bwd_preprocess : D = rowsum(dO * O) (src/attention.py:266), zero dQ_acc
//   bwd main       : per (head, key block, <=128-key slab) item, K_j/V_j
//                    stay on chip; the item's varlen slice is walked in
//                    128-query tiles: gather Q/dO/L/D, recompute S and
//                    P = exp(S - L) (src/attention.py:229), accumulate
//                    dV_j += P^T dO, dK_j += dS^T Q in TMEM
//                    (src/attention.py:230-233); dQ += dS K_j goes to an
//                    fp32 accumulator with bulk reductions
//                    (src/attention.py:234). d = 64: attn_bwd_pipe.cu;
//                    d = 128: moba_bwd_tc_kernel below.
//   bwd_finalize   : dQ = dQ_acc * scale -> bf16 (src/attention.py:299)
#include "common.cuh"
#include "sm100.cuh"
#include <cstdio>
#include <cstdlib>

namespace moba {

constexpr float kLog2eB = 1.4426950408889634f;

// ---------------------------------------------------------------- tcgen05 path
// Persistent CTA per (head, key block, 128-key slab) item, 6 warps:
//   warp 0     producer: K_j / V_j once per item; per 128-query tile the
//              gathered Q, dO rows (cp.async -> mbarrier) and L, D vectors
//   warp 1     MMA issuer: S^T = K Q^T and dP^T = V dO^T (M = keys), then
//              dV += P^T dO, dK += dS^T Q (TMEM accumulators across tiles)
//              and dQ_tile = dS K (M = queries, A operand MN-major)
//   warps 2-5  P^T = exp2(S^T - L), dS^T = P^T (dP^T - D) from TMEM into
//              bf16 SW128 smem tiles; dQ tile TMEM -> fp32 reductions (or
//              per-(query, block) partials); final dK, dV TMEM -> bf16
// TMEM: S^T [0,128) dP^T [128,256) dV [256,256+D) dK [256+D,256+2D),
//       dQ [256+2D, 256+3D) when it fits, else aliased onto S^T.
#define TRACE(slot) do { if (trace && blockIdx.x == 0 && lane == 0 && g < 64) trace[(g) * 16 + (slot)] = clock64(); } while (0)

constexpr int kSmWarps = 8;                               // softmax-bwd warps
constexpr int kPrWarps = 3;                               // producer (gather) warps (16 warps: 128 registers)
constexpr int kMmaWarp = kPrWarps;                        // MMA issuer warp index
constexpr int kSm0 = kPrWarps + 1;                        // first softmax warp
constexpr int kDq0 = kSm0 + kSmWarps;                     // first dQ-epilogue warp
constexpr int kBwdTcThreads = 32 * (kDq0 + 4);

struct BwdBars {
    // a stage's dO half is released after dV (do_empty), its Q half (with the
    // per-row id / L / D vectors) after dK / dQ and the epilogue's id reads
    uint64_t kv_full, kv_empty, q_full[2], q_empty[2], do_full[2], do_empty[2], s_full, p_full, p_empty, pa_full,
        dp_full;
    uint64_t dq_full, dq_empty, dkv_full, dkv_empty;
    uint32_t tmem;
};

template <int D>
__global__ void __launch_bounds__(kBwdTcThreads, 1)
moba_bwd_tc_kernel(const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ dO,
                   const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                   const float* __restrict__ lse, const float* __restrict__ Dd, int64_t N, int B, int width,
                   int kv_group, const int32_t* __restrict__ counts, const int32_t* __restrict__ offsets,
                   const int32_t* __restrict__ flat, float scale, int qstages, int64_t n_items,
                   float* __restrict__ dq_acc, float* __restrict__ dq_part, int64_t part_stride,
                   __nv_bfloat16* __restrict__ dK, __nv_bfloat16* __restrict__ dV, long long* __restrict__ trace) {
    using namespace sm100;
    constexpr int KT = 128;                     // keys per item (M of the key-side MMAs)
    constexpr int MQ = 128;                     // queries per tile
    constexpr bool kDqAlias = (256 + 3 * D > 512);
    constexpr uint32_t kTmemCols = 512;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr uint32_t kv_bytes = KT * D * 2;
    constexpr uint32_t qt_bytes = MQ * D * 2;
    constexpr uint32_t pt_bytes = KT * MQ * 2;
    uint8_t* k_s = smem;
    uint8_t* v_s = k_s + kv_bytes;
    uint8_t* dst_s = v_s + kv_bytes;                 // dS^T  [2 q-slabs][128 keys][128B] (A of dQ)
    uint8_t* stg_s = dst_s + pt_bytes;               // dQ staging: kStgRows rows x (D fp32 + 16 B pad)
    constexpr bool kStage = true;
    // D = 128: 64 staged rows (each epilogue warp stages its 32 rows in two
    // rounds of 16), which fits beside the single Q/dO stage
    constexpr int kStgRows = (D == 64) ? 128 : 64;
    constexpr uint32_t kStgRow = D * 4 + 16;
    uint8_t* stage0 = stg_s + (kStage ? (kStgRows * kStgRow + 1023) / 1024 * 1024 : 0);   // per stage: Q | dO | L | D | qid
    constexpr uint32_t stage_bytes = (2 * qt_bytes + 3 * MQ * 4 + 1023) / 1024 * 1024;  // SW128 tiles need 1 KB alignment
    BwdBars* bars = reinterpret_cast<BwdBars*>(stage0 + qstages * stage_bytes);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n_blocks = (int)((N + B - 1) / B);
    const int slabs = (B + KT - 1) / KT;

    if (warp == kMmaWarp) tmem_alloc(&bars->tmem, kTmemCols);
    if (tid == 0) {
        mbar_init(&bars->kv_full, 1);
        mbar_init(&bars->kv_empty, 1);
        for (int st = 0; st < 2; ++st) {
            mbar_init(&bars->q_full[st], 2 * 32 * kPrWarps);    // cp.async (noinc) + plain arrivals per producer lane
            mbar_init(&bars->do_full[st], 2 * 32 * kPrWarps);
            mbar_init(&bars->q_empty[st], 1 + 4);    // MMA commit + dQ warps (ids read)
            mbar_init(&bars->do_empty[st], 1);       // MMA commit after dV
        }
        mbar_init(&bars->s_full, 1);
        mbar_init(&bars->p_full, kSmWarps);
        mbar_init(&bars->pa_full, kSmWarps);
        mbar_init(&bars->dp_full, 1);
        mbar_init(&bars->p_empty, 1);
        mbar_init(&bars->dq_full, 1);
        mbar_init(&bars->dq_empty, 4);
        mbar_init(&bars->dkv_full, 1);
        mbar_init(&bars->dkv_empty, kSmWarps);
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem;
    // S^T and dP^T swap their 128-column regions every tile: S^T(g+1) goes
    // where dP^T / dS^T(g) were (free once dK(g) has issued), so it no longer
    // waits for the epilogue to drain dQ(g), which aliases S^T(g)'s region;
    // only dP^T(g+1) does
    auto t_s_of = [&](int gg) { return tmem + (uint32_t)(gg & 1) * 128; };
    auto t_dp_of = [&](int gg) { return tmem + (uint32_t)((gg & 1) ^ 1) * 128; };
    const uint32_t t_dv = tmem + 256, t_dk = tmem + 256 + D;
    auto t_dq_of = [&](int gg) { return kDqAlias ? t_s_of(gg) : tmem + 256 + 2 * D; };

    auto stage_ptr = [&](int st) { return stage0 + st * stage_bytes; };

    int g = 0;        // global tile counter (same sequence in every role)
    int kv_use = 0;   // items with >= 1 tile
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int64_t h = item / ((int64_t)n_blocks * slabs);
        const int rem = (int)(item % ((int64_t)n_blocks * slabs));
        const int j = rem / slabs, slab = rem % slabs;
        const int hj = (int)(h * n_blocks + j);
        const int cnt = counts[hj];
        const int n_tiles = (cnt + MQ - 1) / MQ;
        const int64_t kb0 = (int64_t)j * B + slab * KT;
        const int klen = (int)max64(0, min64(min64(KT, (int64_t)B - slab * KT), N - kb0));
        const int32_t* fl = flat + h * N * width + offsets[hj];
        const int64_t pbase = h * N * width + offsets[hj];

        if (warp < kPrWarps) {
            // ------------------------------------------------ producers
            if (warp == 0 && lane == 0 && item == blockIdx.x) {
                tma_prefetch_desc(&tm_k);
                tma_prefetch_desc(&tm_v);
            }
            if (n_tiles > 0 && warp == 0) {
                mbar_wait(&bars->kv_empty, (kv_use & 1) ^ 1);
                if (lane == 0) {
                    mbar_expect_tx(&bars->kv_full, 2 * kv_bytes);
                    const int row0 = (int)((h / kv_group) * N + kb0);   // GQA: K/V head of query head h
#pragma unroll
                    for (int sl = 0; sl < D / 64; ++sl) {
                        tma_load_2d(smem_u32(k_s) + sl * KT * 128, &tm_k, sl * 64, row0, &bars->kv_full);
                        tma_load_2d(smem_u32(v_s) + sl * KT * 128, &tm_v, sl * 64, row0, &bars->kv_full);
                    }
                }
                __syncwarp();
            }
            for (int t = 0; t < n_tiles; ++t, ++g) {
                const int st = g % qstages;
                const int rows = min(MQ, cnt - t * MQ);
                // coalesced gather: 8 lanes cover one 128-B row slab, so a
                // warp instruction touches 4 rows (4 cache lines)
                constexpr int CPR = D / 8;                       // 16-B chunks per row
                const int sub = lane % 8, rsub = lane / 8;
                // warp p gathers rows 4*(p + kPrWarps*i) + rsub
                constexpr int NI = (MQ / 4 + kPrWarps - 1) / kPrWarps;
                int qrow[NI];
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    const int r = 4 * (warp + kPrWarps * i) + rsub;
                    qrow[i] = (r < rows && r < MQ) ? fl[t * MQ + r] : -1;
                }
                // per-row vectors (query id, L, D) of rows 32 (p + kPrWarps i) + l,
                // loaded before the stage wait: their dependent loads (id ->
                // L, D) stay off the gather's critical path
                constexpr int NV = (MQ + 32 * kPrWarps - 1) / (32 * kPrWarps);
                int qv[NV];
                float lv[NV], dv[NV];
#pragma unroll
                for (int i = 0; i < NV; ++i) {
                    const int r = 32 * (warp + kPrWarps * i) + lane;
                    qv[i] = (r < rows && r < MQ) ? fl[t * MQ + r] : -1;
                }
#pragma unroll
                for (int i = 0; i < NV; ++i) {
                    lv[i] = (qv[i] >= 0) ? lse[h * N + qv[i]] * kLog2eB : 0.f;
                    dv[i] = (qv[i] >= 0) ? Dd[h * N + qv[i]] : 0.f;
                }
                const uint32_t qb = smem_u32(stage_ptr(st)), db = qb + qt_bytes;
                const uint32_t l_a = qb + 2 * qt_bytes, d_a = l_a + MQ * 4, id_a = d_a + MQ * 4;
                // dO rows first: their half of the stage frees once dV of the
                // previous tile has run, while phase B and dK / dQ still read Q
                auto gather = [&](uint32_t base, const __nv_bfloat16* src_t) {
#pragma unroll
                    for (int i = 0; i < NI; ++i) {
                        const int r = 4 * (warp + kPrWarps * i) + rsub, qi = qrow[i];
                        if (r >= MQ) continue;
                        const int64_t src = (h * N + max(qi, 0)) * D;
#pragma unroll
                        for (int c = sub; c < CPR; c += 8)
                            cp_async16(base + sw128_off(r, c * 8, MQ), src_t + src + c * 8, qi >= 0);
                    }
                };
                mbar_wait(&bars->do_empty[st], ((g / qstages) & 1) ^ 1);
                gather(db, dO);
                cpasync_arrive_noinc(&bars->do_full[st]);
                mbar_arrive(&bars->do_full[st]);
                mbar_wait(&bars->q_empty[st], ((g / qstages) & 1) ^ 1);
                if (warp == 0) TRACE(0);
                gather(qb, Q);
                cpasync_arrive_noinc(&bars->q_full[st]);
#pragma unroll
                for (int i = 0; i < NV; ++i) {
                    const int r = 32 * (warp + kPrWarps * i) + lane;
                    if (r < MQ) {
                        sts32(id_a + r * 4, (uint32_t)qv[i]);
                        sts32(l_a + r * 4, __float_as_uint(lv[i]));
                        sts32(d_a + r * 4, __float_as_uint(dv[i]));
                    }
                }
                mbar_arrive(&bars->q_full[st]);
                if (warp == 0) TRACE(1);
            }
        } else if (warp == kMmaWarp) {
            // ------------------------------------------------ MMA issuer
            if (n_tiles > 0) mbar_wait(&bars->kv_full, kv_use & 1);
            const uint32_t idesc_kq = idesc_bf16(KT, MQ, false, false);   // S^T, dP^T
            const uint32_t idesc_kd = idesc_bf16(KT, D, false, true);     // dV, dK
            const uint32_t idesc_qd = idesc_bf16(MQ, D, true, true);      // dQ
            const uint32_t kb = smem_u32(k_s), vb = smem_u32(v_s);
            const uint32_t sb = smem_u32(dst_s);
            for (int t = 0; t < n_tiles; ++t, ++g) {
                const int st = g % qstages;
                const uint32_t qb = smem_u32(stage_ptr(st)), db = qb + qt_bytes;
                const uint32_t t_s = t_s_of(g), t_dp = t_dp_of(g);
                mbar_wait(&bars->q_full[st], (g / qstages) & 1);
                TRACE(2);
                tc_fence_after();
                fence_proxy_async_smem();
                // warp-uniform issue (elect.sync inside the asm; a lane-0 region
                // makes the compiler wrap every MMA in an elect/broadcast loop).
                // S^T(g) lands where dS^T(g-1) was: tcgen05.mma runs in issue
                // order, so dK(g-1) has read it by then
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const int sl = kk >> 2, ke = (kk & 3) * 16;
                    umma_bf16_w(t_s, desc_kmajor(kb + sl * KT * 128, ke), desc_kmajor(qb + sl * MQ * 128, ke),
                                idesc_kq, kk > 0);
                }
                umma_commit_w(&bars->s_full);
                TRACE(3);
                // dP^T(g) lands where dQ(g-1) was: wait for its drain
                if (kDqAlias) mbar_wait(&bars->dq_empty, (g & 1) ^ 1);
                mbar_wait(&bars->do_full[st], (g / qstages) & 1);
                tc_fence_after();
                fence_proxy_async_smem();
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const int sl = kk >> 2, ke = (kk & 3) * 16;
                    umma_bf16_w(t_dp, desc_kmajor(vb + sl * KT * 128, ke), desc_kmajor(db + sl * MQ * 128, ke),
                                idesc_kq, kk > 0);
                }
                umma_commit_w(&bars->dp_full);
                if (t == 0) mbar_wait(&bars->dkv_empty, (kv_use & 1) ^ 1);
                // dV += P^T dO as soon as phase A has stored P^T (runs under phase B)
                mbar_wait(&bars->pa_full, g & 1);
                TRACE(4);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < MQ / 16; ++kk) {
                    const uint32_t acol = 64 * (kk >> 2) + 8 * (kk & 3);
                    umma_bf16_ts_w(t_dv, t_s + acol, desc_mnmajor(db, kk * 16, MQ * 128), idesc_kd, (t > 0) || (kk > 0));
                }
                umma_commit_w(&bars->do_empty[st]);      // dP^T and dV have read dO
                mbar_wait(&bars->p_full, g & 1);
                if (!kDqAlias) mbar_wait(&bars->dq_empty, (g & 1) ^ 1);
                TRACE(5);
                tc_fence_after();
                fence_proxy_async_smem();
                // dK += dS^T Q   (K = queries; dS^T bf16 in TMEM)
#pragma unroll
                for (int kk = 0; kk < MQ / 16; ++kk) {
                    const uint32_t acol = 64 * (kk >> 2) + 8 * (kk & 3);
                    umma_bf16_ts_w(t_dk, t_dp + acol, desc_mnmajor(qb, kk * 16, MQ * 128), idesc_kd, (t > 0) || (kk > 0));
                }
                // dQ_tile = dS K   (M = queries from dS^T as MN-major A, K = keys),
                // over S^T(g) / P^T(g) (read by phase A and the dV MMAs above)
#pragma unroll
                for (int kk = 0; kk < KT / 16; ++kk)
                    umma_bf16_w(t_dq_of(g), desc_mnmajor(sb, kk * 16, KT * 128), desc_mnmajor(kb, kk * 16, KT * 128),
                                idesc_qd, kk > 0);
                umma_commit_w(&bars->dq_full);
                umma_commit_w(&bars->p_empty);
                umma_commit_w(&bars->q_empty[st]);
                if (t + 1 == n_tiles) {
                    umma_commit_w(&bars->dkv_full);
                    umma_commit_w(&bars->kv_empty);
                }
            }
        } else if (warp < kDq0) {
            // ------------------------------------------------ softmax-bwd (8 warps)
            // warp pair (w, w+4) shares TMEM lane quadrant w&3; `half` picks
            // the query columns [64*half, 64*half+64) of S^T / dP^T
            const int quad = warp & 3;
            const int half = (warp - kSm0) >> 2;
            const int row = 32 * quad + lane;                     // key row
            const uint32_t lane_off = (uint32_t)(32 * quad) << 16;
            const int64_t key = kb0 + row;
            const bool krow_ok = row < klen;
            const float sl2 = kLog2eB * scale;
            const uint32_t ds_a = smem_u32(dst_s);
            for (int t = 0; t < n_tiles; ++t, ++g) {
                const int st = g % qstages;
                const uint32_t l_a = smem_u32(stage_ptr(st)) + 2 * qt_bytes, d_a = l_a + MQ * 4, id_a = d_a + MQ * 4;
                const uint32_t t_s = t_s_of(g), t_dp = t_dp_of(g);
                mbar_wait(&bars->s_full, g & 1);
                if (warp == kSm0) TRACE(6);
                tc_fence_after();
                const int rows_t = min(MQ, cnt - t * MQ);
                // tile-uniform: slices are ascending, so if the first query is
                // at or past the slab's last key no element of the tile is masked
                const bool need_mask = rows_t < MQ || klen < KT || (int64_t)lds32i(id_a) < kb0 + KT - 1;
                // padded rows carry id -1, dead key rows never pass
                const int kmask = krow_ok ? (int)key : 0x7fffffff;
                // phase A: P = exp2(S^T scale log2e - L) kept in fp32 for phase
                // B; bf16 pairs over the S^T columns just read (A of dV).
                // The mask test is a template argument, not a branch inside
                // the unrolled loop (per-group branches serialise the loads
                // and exponentials)
                float pv[64];
                auto phase_a = [&](auto mask_tag) {
                    constexpr bool kMask = decltype(mask_tag)::value;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int c0 = half * 64 + c * 16;
                        float sv[16];
                        tmem_ld16(t_s + lane_off + c0, sv);
                        tmem_ld_wait();
                        uint32_t pk[8];
#pragma unroll
                        for (int i = 0; i < 16; i += 4) {
                            const float4 lv = lds128f(l_a + (c0 + i) * 4);
                            const float la[4] = {lv.x, lv.y, lv.z, lv.w};
                            float* p4 = &pv[c * 16 + i];
                            if constexpr (kMask) {
                                const int4 iv = lds128i(id_a + (c0 + i) * 4);
                                const int ia[4] = {iv.x, iv.y, iv.z, iv.w};
#pragma unroll
                                for (int u = 0; u < 4; ++u) {
                                    const float e = fast_exp2(fmaf(sv[i + u], sl2, -la[u]));
                                    p4[u] = kmask <= ia[u] ? e : 0.f;
                                }
                            } else {
#pragma unroll
                                for (int u = 0; u < 4; ++u) p4[u] = fast_exp2(fmaf(sv[i + u], sl2, -la[u]));
                            }
                            pk[i >> 1] = pack_bf16(p4[0], p4[1]);
                            pk[(i >> 1) + 1] = pack_bf16(p4[2], p4[3]);
                        }
                        tmem_st8(t_s + lane_off + half * 64 + c * 8, pk);
                    }
                };
                if (need_mask)
                    phase_a(std::true_type{});
                else
                    phase_a(std::false_type{});
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->pa_full);
                // phase B: dS^T = P (dP^T - D) -> bf16 pairs over the dP^T
                // columns (A of dK) and the SW128 smem tile (A of dQ), which
                // the dQ MMA of the previous tile has finished reading (p_empty)
                mbar_wait(&bars->p_empty, (g & 1) ^ 1);
                mbar_wait(&bars->dp_full, g & 1);
                if (warp == kSm0) TRACE(7);
                tc_fence_after();
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int c0 = half * 64 + c * 16;
                    float dpv[16];
                    tmem_ld16(t_dp + lane_off + c0, dpv);
                    tmem_ld_wait();
                    uint32_t dk[8];
#pragma unroll
                    for (int i = 0; i < 16; i += 4) {
                        const float4 dv = lds128f(d_a + (c0 + i) * 4);
                        const float da[4] = {dv.x, dv.y, dv.z, dv.w};
                        const float* p4 = &pv[c * 16 + i];
                        dk[i >> 1] = pack_bf16(p4[0] * (dpv[i] - da[0]), p4[1] * (dpv[i + 1] - da[1]));
                        dk[(i >> 1) + 1] = pack_bf16(p4[2] * (dpv[i + 2] - da[2]), p4[3] * (dpv[i + 3] - da[3]));
                    }
                    tmem_st8(t_dp + lane_off + half * 64 + c * 8, dk);
#pragma unroll
                    for (int gq = 0; gq < 2; ++gq) {
                        const uint32_t off = sw128_off(row, c0 + gq * 8, KT);
                        sts128(ds_a + off, make_uint4(dk[4 * gq], dk[4 * gq + 1], dk[4 * gq + 2], dk[4 * gq + 3]));
                    }
                }
                tmem_st_wait();
                tc_fence_before();
                fence_proxy_async_smem();
                __syncwarp();
                if (warp == kSm0) TRACE(8);
                if (lane == 0) mbar_arrive(&bars->p_full);
            }
            // ---- dK, dV of this slab (zeros when no query attends); D split by half
            if (n_tiles > 0) {
                mbar_wait(&bars->dkv_full, kv_use & 1);
                tc_fence_after();
            }
#pragma unroll
            for (int cc = 0; cc < D / 64; ++cc) {
                const int c0 = half * (D / 2) + cc * 32;
                float kv[32], vv[32];
                if (n_tiles > 0) {
                    tmem_ld32(t_dk + lane_off + c0, kv);
                    tmem_ld32(t_dv + lane_off + c0, vv);
                    tmem_ld_wait();
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) kv[i] = vv[i] = 0.f;
                }
                if (row < klen) {
                    uint32_t pk[16], pv[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        pk[i] = pack_bf16(kv[2 * i] * scale, kv[2 * i + 1] * scale);
                        pv[i] = pack_bf16(vv[2 * i], vv[2 * i + 1]);
                    }
                    const int64_t o = (h * N + key) * D + c0;
#pragma unroll
                    for (int gq = 0; gq < 4; ++gq) {
                        *reinterpret_cast<uint4*>(dK + o + gq * 8) = make_uint4(pk[4 * gq], pk[4 * gq + 1], pk[4 * gq + 2], pk[4 * gq + 3]);
                        *reinterpret_cast<uint4*>(dV + o + gq * 8) = make_uint4(pv[4 * gq], pv[4 * gq + 1], pv[4 * gq + 2], pv[4 * gq + 3]);
                    }
                }
            }
            if (n_tiles > 0) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->dkv_empty);
            }
        } else {
            // ------------------------------------------------ dQ epilogue (4 warps)
            const int quad = warp & 3;
            const int row = 32 * quad + lane;                     // query row of the tile
            const uint32_t lane_off = (uint32_t)(32 * quad) << 16;
            for (int t = 0; t < n_tiles; ++t, ++g) {
                const int st = g % qstages;
                const uint32_t id_a = smem_u32(stage_ptr(st)) + 2 * qt_bytes + 2 * MQ * 4;
                mbar_wait(&bars->dq_full, g & 1);
                if (warp == kDq0) TRACE(9);
                tc_fence_after();
                const int qi = lds32i(id_a + row * 4);
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->q_empty[st]);    // ids read: the Q half may be refilled
                const int r_in = t * MQ + row;
                if constexpr (!kStage) {
                    // no room for a staging buffer: vector reductions straight from registers
#pragma unroll
                    for (int c0 = 0; c0 < D; c0 += 32) {
                        float v[32];
                        tmem_ld32(t_dq_of(g) + lane_off + c0, v);
                        tmem_ld_wait();
                        if (qi >= 0) {
                            if (dq_part != nullptr) {
                                float* dst = dq_part + slab * part_stride + (pbase + r_in) * D + c0;
#pragma unroll
                                for (int i = 0; i < 32; i += 4)
                                    *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                            } else {
                                float* dst = dq_acc + (h * N + qi) * D + c0;
#pragma unroll
                                for (int i = 0; i < 32; i += 4) red_add_f32x4(dst + i, v[i], v[i + 1], v[i + 2], v[i + 3]);
                            }
                        }
                    }
                } else if constexpr (D == 128) {
                    // two rounds of 16 lanes over 16 staged rows per warp; every
                    // lane takes part in the (warp-collective) TMEM loads
                    const uint32_t srow = smem_u32(stg_s) + (quad * 16 + (lane & 15)) * kStgRow;
#pragma unroll
                    for (int rr = 0; rr < 2; ++rr) {
                        bulk_wait_read0();               // this lane's previous bulk op has read its row
                        __syncwarp();
                        const bool mine = (lane >> 4) == rr;
#pragma unroll
                        for (int c0 = 0; c0 < D; c0 += 32) {
                            float v[32];
                            tmem_ld32(t_dq_of(g) + lane_off + c0, v);
                            tmem_ld_wait();
                            if (mine) {
#pragma unroll
                                for (int i = 0; i < 32; i += 4)
                                    sts128(srow + (c0 + i) * 4,
                                           make_uint4(__float_as_uint(v[i]), __float_as_uint(v[i + 1]),
                                                      __float_as_uint(v[i + 2]), __float_as_uint(v[i + 3])));
                            }
                        }
                        if (mine) {
                            fence_proxy_async_smem();
                            if (qi >= 0) {
                                if (dq_part != nullptr)
                                    bulk_store(dq_part + slab * part_stride + (pbase + r_in) * D, srow, D * 4);
                                else
                                    bulk_reduce_add_f32(dq_acc + (h * N + qi) * D, srow, D * 4);
                            }
                            bulk_commit();
                        }
                    }
                } else {
                // TMEM -> padded fp32 staging row -> one bulk reduce (or store) per row
                const uint32_t srow = smem_u32(stg_s) + row * kStgRow;
                bulk_wait_read0();                       // previous tile's bulk ops have read the row
#pragma unroll
                for (int c0 = 0; c0 < D; c0 += 32) {
                    float v[32];
                    tmem_ld32(t_dq_of(g) + lane_off + c0, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; i += 4)
                        sts128(srow + (c0 + i) * 4, make_uint4(__float_as_uint(v[i]), __float_as_uint(v[i + 1]),
                                                               __float_as_uint(v[i + 2]), __float_as_uint(v[i + 3])));
                }
                fence_proxy_async_smem();
                if (qi >= 0) {
                    if (dq_part != nullptr)
                        bulk_store(dq_part + slab * part_stride + (pbase + r_in) * D, srow, D * 4);
                    else
                        bulk_reduce_add_f32(dq_acc + (h * N + qi) * D, srow, D * 4);
                }
                bulk_commit();
                }
                tc_fence_before();
                __syncwarp();
                if (warp == kDq0) TRACE(10);
                if (lane == 0) mbar_arrive(&bars->dq_empty);
            }
        }
        if (n_tiles > 0) ++kv_use;
    }
    if (warp >= kDq0) bulk_wait0();
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc(tmem, kTmemCols);
    }
}

// D = rowsum(dO * O) and dq_acc = 0; one warp per row.
template <int D>
// D = rowsum(dO * O) (src/attention.py:266) and dQ accumulator zeroing:
// D/8 lanes per row, 16-B loads and stores, 32/(D/8) rows per warp.
__global__ void bwd_preprocess_kernel(const __nv_bfloat16* __restrict__ O, const __nv_bfloat16* __restrict__ dO,
                                      int64_t rows, float* __restrict__ Dd, float* __restrict__ dq_acc) {
    constexpr int L = D / 8, G = 32 / L;
    const int lane = threadIdx.x & 31, grp = lane / L, sub = lane % L;
    const int64_t row = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * G + grp;
    const bool ok = row < rows;
    const int64_t r = ok ? row : 0;
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(O + r * D) + sub);
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(dO + r * D) + sub);
    const uint32_t ua[4] = {a.x, a.y, a.z, a.w}, ub[4] = {b.x, b.y, b.z, b.w};
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const float2 x = unpack_bf16(ua[c]), y = unpack_bf16(ub[c]);
        s = fmaf(x.x, y.x, fmaf(x.y, y.y, s));
    }
#pragma unroll
    for (int o = 1; o < L; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (ok) {
        if (sub == 0) Dd[row] = s;
        float4* z = reinterpret_cast<float4*>(dq_acc + row * D + sub * 8);
        z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
        z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

__global__ void bwd_finalize_kernel(const float* __restrict__ dq_acc, int64_t n, float scale,
                                    __nv_bfloat16* __restrict__ dQ) {
    const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
    if (e >= n) return;
    const float4 v = __ldg(reinterpret_cast<const float4*>(dq_acc + e));
    const float4 w = __ldg(reinterpret_cast<const float4*>(dq_acc + e) + 1);
    *reinterpret_cast<uint4*>(dQ + e) = make_uint4(pack_bf16(v.x * scale, v.y * scale), pack_bf16(v.z * scale, v.w * scale),
                                                   pack_bf16(w.x * scale, w.y * scale), pack_bf16(w.z * scale, w.w * scale));
}

// deterministic dQ: per query, sum its partials in (slot, slab) order.
// Deterministic dQ: a query's fp32 per-(query, block) partial rows summed in
// slot order (fixed order -> bitwise reproducible). L = D/4 lanes per query
// (16 B of the fp32 row each): 2 queries per warp at d = 64, 1 at d = 128;
// the group's lanes load the positions of slots sub, sub + L, ... and
// broadcast them, and every partial row of a batch of up to 16 slots is in
// flight before any is added.
template <int D, int W>
__global__ void __launch_bounds__(128)
bwd_dq_combine_kernel(const float* __restrict__ dq_part, int64_t part_stride, int slabs,
                      const int32_t* __restrict__ row_pos, int64_t N, int width, int64_t rows, float scale,
                      __nv_bfloat16* __restrict__ dQ) {
    constexpr int L = D / 4;                  // lanes per query
    constexpr int QPW = 32 / L;
    constexpr int C = (W + L - 1) / L;
    constexpr int NB = W < 16 ? W : 16;
    const int lane = threadIdx.x & 31, grp = lane / L, sub = lane % L, g0 = grp * L;
    const int64_t row = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * QPW + grp;
    const bool ok = row < rows;
    const int64_t r = ok ? row : rows - 1;
    const int64_t h = rows < (1ll << 31) ? (int64_t)((uint32_t)r / (uint32_t)N) : r / N;
    int32_t p[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int sl = sub + L * c;
        p[c] = (sl < width) ? __ldg(row_pos + r * width + sl) : -1;
    }
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int sb = 0; sb < slabs; ++sb) {
        const float4* base = reinterpret_cast<const float4*>(dq_part + sb * part_stride + h * N * width * D) + sub;
#pragma unroll
        for (int v0 = 0; v0 < W; v0 += NB) {
            if (v0 >= width) break;
            float4 x[NB];
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                const int v = v0 + u;
                const int32_t pv = __shfl_sync(0xffffffffu, p[v / L], g0 + v % L);
                x[u] = (v < width && pv >= 0) ? __ldg(base + (int64_t)pv * (D / 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                acc.x += x[u].x;
                acc.y += x[u].y;
                acc.z += x[u].z;
                acc.w += x[u].w;
            }
        }
    }
    if (!ok) return;
    *reinterpret_cast<uint2*>(dQ + row * D + sub * 4) =
        make_uint2(pack_bf16(acc.x * scale, acc.y * scale), pack_bf16(acc.z * scale, acc.w * scale));
}

int launch_bwd_pipe(const void* q, const void* k, const void* v, const void* dout, const float* lse, const float* Dd,
                    int64_t bh, int kv_group, int64_t N, int B, int width, const int32_t* counts, const int32_t* offsets,
                    const int32_t* flat, float scale, int* sched, float* dq_acc, float* dq_part,
                    int64_t part_stride, void* dk, void* dv, cudaStream_t s);

// workspace: sched int (256 B) | Dd f32 [bh*N] | dq_acc f32 [bh*N*D] |
// (deterministic) dq_part f32 [slabs][bh*N*width*D]
static size_t bwd_ws(int64_t bh, int64_t N, int D, int B, int width, bool det, int kv_group = 1) {
    size_t w = 256 + align_up((size_t)bh * N * 4, 256) + align_up((size_t)bh * N * D * 4, 256);
    if (det) w += (size_t)ceil_div(B, 128) * bh * N * width * D * 4;
    if (kv_group > 1) w += 2 * align_up((size_t)bh * N * D * 2, 256);   // per-query-head dK, dV (bf16)
    return w;
}

// GQA: dK/dV of a K/V head = sum over its kv_group query heads (fp32 sum of
// the per-query-head bf16 gradients, fixed order -> deterministic)
__global__ void gqa_group_sum_kernel(const __nv_bfloat16* __restrict__ src, int64_t kv_rows_elems, int64_t head_elems,
                                     int kv_group, __nv_bfloat16* __restrict__ dst) {
    const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
    if (e >= kv_rows_elems) return;
    const int64_t hk = e / head_elems, off = e - hk * head_elems;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int g = 0; g < kv_group; ++g) {
        const uint4 u = *reinterpret_cast<const uint4*>(src + (hk * kv_group + g) * head_elems + off);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const float2 f = unpack_bf16(w[c]);
            acc[2 * c] += f.x;
            acc[2 * c + 1] += f.y;
        }
    }
    *reinterpret_cast<uint4*>(dst + e) = make_uint4(pack_bf16(acc[0], acc[1]), pack_bf16(acc[2], acc[3]),
                                                    pack_bf16(acc[4], acc[5]), pack_bf16(acc[6], acc[7]));
}

template <int D>
static int launch_bwd(const void* q, const void* k, const void* v, const void* out, const void* dout,
                      const float* lse, int64_t bh, int kv_group, int64_t N, int B, int width, const int32_t* counts,
                      const int32_t* offsets, const int32_t* flat, const int32_t* row_pos, bool det, float scale,
                      void* dq, void* dk_out, void* dv_out, uint8_t* ws, cudaStream_t s) {
    int* sched = (int*)ws;
    ws += 256;
    float* Dd = (float*)ws;
    float* dq_acc = (float*)(ws + align_up((size_t)bh * N * 4, 256));
    float* dq_part = det ? (float*)((uint8_t*)dq_acc + align_up((size_t)bh * N * D * 4, 256)) : nullptr;
    const int64_t part_stride = bh * N * width * D;
    const int slabs = (int)ceil_div(B, 128);
    const int64_t rows = bh * N;
    // GQA: the kernels write per-query-head dK / dV, summed per group below
    void* dk = dk_out;
    void* dv = dv_out;
    if (kv_group > 1) {
        uint8_t* g = (uint8_t*)dq_acc + align_up((size_t)bh * N * D * 4, 256) +
                     (det ? (size_t)slabs * bh * N * width * D * 4 : 0);
        dk = g;
        dv = g + align_up((size_t)bh * N * D * 2, 256);
    }
    {
    StageTimer tm(T_BWD_PRE, s);
    bwd_preprocess_kernel<D><<<(unsigned)ceil_div(rows, 8 * (256 / D)), 256, 0, s>>>((const __nv_bfloat16*)out,
                                                                        (const __nv_bfloat16*)dout, rows, Dd, dq_acc);
    }
    int st = check_launch("bwd_preprocess_kernel");
    if (st) return st;
    {
    StageTimer tm(T_BWD, s);
    if (D == 64) {
        // pipelined tcgen05 kernel (attn_bwd_pipe.cu); dq_part slabs follow its 128-key slabs
        st = launch_bwd_pipe(q, k, v, dout, lse, Dd, bh, kv_group, N, B, width, counts, offsets, flat, scale, sched,
                             dq_acc, dq_part, part_stride, dk, dv, s);
    } else {
        const size_t stage_bytes = align_up(2 * (size_t)128 * D * 2 + 3 * 128 * 4, 1024);
        const size_t stg_bytes = align_up((size_t)(D == 64 ? 128 : 64) * (D * 4 + 16), 1024);
        const size_t fixed = 1024 + 2 * (size_t)128 * D * 2 + (size_t)128 * 128 * 2 + stg_bytes + sizeof(BwdBars);
        const int qstages = (fixed + 2 * stage_bytes <= 232448) ? 2 : 1;
        const size_t smem = fixed + qstages * stage_bytes;
        if (smem > 232448) return MOBA_ERR_UNSUPPORTED;
        // debug timeline (MOBA_TRACE): a kernel argument, so a captured graph
        // holds no host-memory copy node
        static long long* tr = nullptr;
        const bool tracing = std::getenv("MOBA_TRACE") != nullptr;
        if (tracing) {
            if (!tr) cudaMalloc(&tr, 64 * 16 * 8);
            cudaMemsetAsync(tr, 0, 64 * 16 * 8, s);
        }
        long long* trp = tracing ? tr : nullptr;
        CUtensorMap tm_k, tm_v;
        if (!make_tmap_bf16(&tm_k, k, (uint64_t)(bh / kv_group * N), D, 128) ||
            !make_tmap_bf16(&tm_v, v, (uint64_t)(bh / kv_group * N), D, 128))
            return MOBA_ERR_CUDA;
        auto kern = moba_bwd_tc_kernel<D>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int64_t n_items = bh * ceil_div(N, B) * ceil_div(B, 128);
        const int grid = (int)std::min<int64_t>(n_items, kNumSMs);
        kern<<<grid, kBwdTcThreads, smem, s>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)dout, tm_k, tm_v, lse, Dd, N, B,
                                               width, kv_group, counts, offsets, flat, scale, qstages, n_items, dq_acc,
                                               dq_part, part_stride, (__nv_bfloat16*)dk, (__nv_bfloat16*)dv, trp);
        st = check_launch("moba_bwd_tc_kernel");
        if (st == 0 && tracing) {
            static long long host[64 * 16];
            cudaMemcpyAsync(host, tr, sizeof(host), cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            if (FILE* f = std::fopen(std::getenv("MOBA_TRACE"), "wb")) {
                std::fwrite(host, sizeof(host), 1, f);
                std::fclose(f);
            }
        }
    }
    }
    if (st) return st;
    StageTimer tm(T_BWD_POST, s);
    if (kv_group > 1) {
        const int64_t kv_elems = bh / kv_group * N * D;
        for (int which = 0; which < 2; ++which)
            gqa_group_sum_kernel<<<(unsigned)ceil_div(kv_elems / 8, 256), 256, 0, s>>>(
                (const __nv_bfloat16*)(which ? dv : dk), kv_elems, N * D, kv_group,
                (__nv_bfloat16*)(which ? dv_out : dk_out));
        st = check_launch("gqa_group_sum_kernel", 2);
        if (st) return st;
    }
    if (det) {
        const unsigned grid = (unsigned)ceil_div(rows, 4 * (128 / D));   // 4 warps x (32 / (D / 4)) queries
#define MOBA_DQC(W) bwd_dq_combine_kernel<D, W><<<grid, 128, 0, s>>>(dq_part, part_stride, slabs, row_pos, N, width, \
                                                                     rows, scale, (__nv_bfloat16*)dq)
        if (width <= 4) MOBA_DQC(4);
        else if (width <= 8) MOBA_DQC(8);
        else if (width <= 9) MOBA_DQC(9);
        else if (width <= 16) MOBA_DQC(16);
        else if (width <= 17) MOBA_DQC(17);
        else MOBA_DQC(32);
#undef MOBA_DQC
        return check_launch("bwd_dq_combine_kernel");
    }
    const int64_t ne = rows * D;
    bwd_finalize_kernel<<<(unsigned)ceil_div(ne / 8, 256), 256, 0, s>>>(dq_acc, ne, scale, (__nv_bfloat16*)dq);
    return check_launch("bwd_finalize_kernel");
}

}  // namespace moba

using namespace moba;

extern "C" size_t moba_bwd_gqa_workspace_size(int64_t bh, int kv_group, int64_t n_tokens, int head_dim,
                                              int block_size, int width, int deterministic) {
    if (bh < 1 || n_tokens < 1 || block_size < 1 || width < 1 || kv_group < 1) return 0;
    return bwd_ws(bh, n_tokens, head_dim, block_size, width, deterministic != 0, kv_group);
}

extern "C" size_t moba_bwd_workspace_size(int64_t bh, int64_t n_tokens, int head_dim, int block_size, int width,
                                          int deterministic) {
    return moba_bwd_gqa_workspace_size(bh, 1, n_tokens, head_dim, block_size, width, deterministic);
}

extern "C" int moba_bwd_gqa(const void* q, const void* k, const void* v, const void* out, const void* dout,
                            const float* lse, int64_t bh, int kv_group, int64_t n_tokens, int head_dim, int block_size,
                            int width, const int32_t* counts, const int32_t* offsets, const int32_t* flat,
                            const int32_t* row_pos, int deterministic, float softmax_scale, void* dq, void* dk,
                            void* dv, void* workspace, size_t workspace_bytes, void* stream) {
    clear_last_error();
    if (bh < 1 || bh > 65535 || n_tokens < 1 || block_size < 1 || width < 1) return MOBA_ERR_SHAPE;
    if (kv_group < 1 || bh % kv_group != 0) return MOBA_ERR_SHAPE;
    if (block_size > 512 || width > 32) return MOBA_ERR_UNSUPPORTED;
    const bool det = deterministic != 0;
    if (det && row_pos == nullptr) return MOBA_ERR_PLAN;
    if (workspace_bytes < bwd_ws(bh, n_tokens, head_dim, block_size, width, det, kv_group)) return MOBA_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t* ws = (uint8_t*)workspace;
    if (head_dim == 64)
        return launch_bwd<64>(q, k, v, out, dout, lse, bh, kv_group, n_tokens, block_size, width, counts, offsets,
                              flat, row_pos, det, softmax_scale, dq, dk, dv, ws, s);
    if (head_dim == 128)
        return launch_bwd<128>(q, k, v, out, dout, lse, bh, kv_group, n_tokens, block_size, width, counts, offsets,
                               flat, row_pos, det, softmax_scale, dq, dk, dv, ws, s);
    return MOBA_ERR_UNSUPPORTED;
}

extern "C" int moba_bwd(const void* q, const void* k, const void* v, const void* out, const void* dout,
                        const float* lse, int64_t bh, int64_t n_tokens, int head_dim, int block_size, int width,
                        const int32_t* counts, const int32_t* offsets, const int32_t* flat, const int32_t* row_pos,
                        int deterministic, float softmax_scale, void* dq, void* dk, void* dv, void* workspace,
                        size_t workspace_bytes, void* stream) {
    return moba_bwd_gqa(q, k, v, out, dout, lse, bh, 1, n_tokens, head_dim, block_size, width, counts, offsets, flat,
                        row_pos, deterministic, softmax_scale, dq, dk, dv, workspace, workspace_bytes, stream);
}
